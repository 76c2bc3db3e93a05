"""B200-native pipelined two-stage FP64 symmetric EVD (arXiv 2511.16174), drop-in for `pipeevd`."""
__version__ = "0.1.0"

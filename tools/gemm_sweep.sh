P=tools/kernel_probe.py
for c in 0 1 2 3 4; do
  echo "cfg $c"
  for s in "8192 8192 8192" "8192 8192 8192 1 0" "8192 8192 8192 0 1" "512 49152 24576 1 0" "24576 49152 512" "24576 24576 256 0 1"; do
    PEVD_GEMM=$c timeout 60 python $P gemm $s
  done
done

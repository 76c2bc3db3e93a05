"""`python -m paper_2511_16174_b200 ...` runs the command-line front end (cli.py)."""
import sys

from .cli import main

sys.exit(main())

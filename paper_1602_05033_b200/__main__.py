"""``python -m paper_1602_05033_b200 ...``: the command line (cli.py)."""
import sys

from .cli import main

sys.exit(main())

"""`python -m paper_1905_10574_b200 ...`: the rsylv-bench CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())

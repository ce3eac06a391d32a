"""`python -m paper_2510_03426_b200 ...`: the command-line front end (cli.py)."""
import sys

from .cli import main

sys.exit(main())

"""`python -m paper_1309_1889_b200 <gen|simulate|compare|parareal> ...` (cli.py)."""
import sys

from .cli import main

sys.exit(main())

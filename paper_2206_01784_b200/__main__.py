"""`python -m paper_2206_01784_b200 gen|sort|verify|bench ...` (cli.py)."""

import sys

from .cli import main

sys.exit(main())

"""`python -m paper_2106_06889_b200 analyze|verify|bench ...` (see cli.py)."""

import sys

from .cli import main

sys.exit(main())

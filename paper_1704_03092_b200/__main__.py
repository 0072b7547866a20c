"""`python -m paper_1704_03092_b200 ...`: the benchmark front end (cli.py)."""

import sys

from .cli import main

sys.exit(main())

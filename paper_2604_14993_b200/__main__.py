"""``python -m paper_2604_14993_b200 compose|simulate ...`` (see cli.py)."""

import sys

from .cli import main

sys.exit(main())

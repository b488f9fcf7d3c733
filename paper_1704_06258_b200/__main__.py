"""python -m paper_1704_06258_b200 <command> (see cli.py)."""

import sys

from .cli import main

sys.exit(main())

"""``python -m paper_2605_14419_b200 {sort,verify} ...`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())

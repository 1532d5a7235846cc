"""``python -m paper_2110_01470_b200 run|sweep ...`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())

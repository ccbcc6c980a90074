"""python -m paper_2008_02734_b200 {align,compare,memreport} ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())

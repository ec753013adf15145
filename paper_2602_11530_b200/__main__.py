"""python -m paper_2602_11530_b200 gen|run|sweep|compare (see cli.py)."""
import sys

from .cli import main

sys.exit(main())

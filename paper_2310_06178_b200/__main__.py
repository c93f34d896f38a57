"""python -m paper_2310_06178_b200 <command> ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())

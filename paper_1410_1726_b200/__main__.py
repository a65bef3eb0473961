"""python -m paper_1410_1726_b200 run ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())

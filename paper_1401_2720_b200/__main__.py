"""python -m paper_1401_2720_b200 ... (the reference CLI, cli.py)."""
import sys

from .cli import main

sys.exit(main())

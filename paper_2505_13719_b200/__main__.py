"""python -m paper_2505_13719_b200 solve ... (cli.py)."""
import sys

from .cli import main

sys.exit(main())

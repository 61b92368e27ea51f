"""``python -m paper_2511_10442_b200 <gen|knn|verify|ochelper> ...`` (cli.py)."""
import sys

from .cli import main

sys.exit(main())

"""``python -m paper_2201_12465_b200 bench ...`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())

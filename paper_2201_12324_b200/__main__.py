"""``python -m paper_2201_12324_b200 lin ...`` (see cli.py)."""

import sys

from .cli import main

sys.exit(main())

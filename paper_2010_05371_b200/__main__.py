"""python -m paper_2010_05371_b200 == the CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())

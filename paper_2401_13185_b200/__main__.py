"""`python -m paper_2401_13185_b200 {verify,run,bench}` — see cli.py."""
import sys

from .cli import main

sys.exit(main())

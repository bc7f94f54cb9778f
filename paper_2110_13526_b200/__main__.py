"""python -m paper_2110_13526_b200 <command> ...  (see cli.py)."""
from .cli import entry

entry()

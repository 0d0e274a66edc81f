"""python -m paper_2105_07544_b200 {solve,generate,sweep-switch,sweep-restart} ..."""
from .cli import entry

entry()

"""python -m mpkrylov ... -> the GPU-backed CLI (paper_2105_07544_b200.cli)."""
from mpkrylov.cli import entry

entry()

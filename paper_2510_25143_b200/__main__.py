"""python -m paper_2510_25143_b200 ... : the CLI (cli.py)."""
from .cli import main

main()

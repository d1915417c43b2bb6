"""`python -m paper_2509_06971_b200 run ...` -- the reference's `petto run` on the B200 (cli.py)."""
import sys

from .cli import main

sys.exit(main())

"""`python -m paper_2007_14178_b200 {bench,conv,verify}` (the reference's `xnorconv` script)."""
import sys

from .cli import main

sys.exit(main())

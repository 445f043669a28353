"""``python -m paper_1402_3789_b200 <cluster|generate|bench> ...`` (cli.main)."""

import sys

from .cli import main

sys.exit(main())

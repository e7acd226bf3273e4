"""``python -m kltune`` — the reference's ``kltune`` console script
(reference pkg/pyproject.toml:20-21 -> kltune.cli:main) on the B200 package."""

import sys

from paper_2303_12374_b200.cli import main

sys.exit(main())

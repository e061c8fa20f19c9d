"""``python -m paper_0911_3456_b200`` runs the ``rtcg`` command line."""

import sys

from .cli import main

sys.exit(main())

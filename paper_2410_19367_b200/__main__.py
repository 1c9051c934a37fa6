"""``python -m paper_2410_19367_b200 <plan|compare|simulate|search|render|verify> ...``
(the reference's declared ``pipesched`` console script, pkg/pyproject.toml:19-20)."""
import sys

from .cli import main

sys.exit(main())

"""CPU oracle for the GBS hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  The product path
(paper_2501_13382_b200) never imports it and fails loudly without its CUDA
library.
"""
from .oracle import (build, gbs_accumulate, load_bundle, nearest_on_segments,  # noqa: F401
                     trace, worklist)

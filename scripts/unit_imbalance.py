"""Per-unit cycle counts (BF_UNIT_TIMES build) -> how unevenly the 8 patches of a tile
share a beam range: sum over (tile, range) of max / mean over its patch units.
    python scripts/unit_imbalance.py unit_cycles.bin"""
import sys

import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.int64)
n_patches, n_ranges, ppt = (int(v) for v in raw[:3])
cyc = raw[3:].reshape(n_ranges, n_patches).astype(np.float64)
n_tiles = (n_patches + ppt - 1) // ppt
pad = n_tiles * ppt - n_patches
c = np.concatenate([cyc, np.zeros((n_ranges, pad))], axis=1).reshape(n_ranges, n_tiles, ppt)
tot = c.sum()
mx = c.max(axis=2).sum() * ppt
print(f"units {n_patches * n_ranges}, total cycles {tot:.3e}; if the {ppt} patches of a tile "
      f"ran in lockstep per range: {mx:.3e} ({mx / tot:.2f}x)")

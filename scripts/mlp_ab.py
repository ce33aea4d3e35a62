"""A/B of two MLP kernel variants selected by an environment switch: identical
outputs (bit for bit) over several batch sizes.   python scripts/mlp_ab.py VAR rows..."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2104_13542_b200.surrogate import load_arm7_surrogate  # noqa: E402

var = sys.argv[1]
m = load_arm7_surrogate()
for rows in [int(a) for a in sys.argv[2:]] or [1000, 100_000, 1_000_003]:
    q = np.random.default_rng(rows).uniform(-3, 3, size=(rows, 7))
    outs = []
    for v in ("0", "1"):
        os.environ[var] = v
        outs.append(m.distance(q))
    d = np.abs(outs[0] - outs[1])
    print(f"rows {rows}: max |a - b| = {d.max():.3e} ({(d > 0).sum()} differ)", flush=True)

"""Two-slot MLP (mlp2_tcgen05_kernel) vs the one-tile kernel: bit-identical
outputs over several batch sizes (and v2 run-to-run determinism)."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2104_13542_b200.surrogate import load_arm7_surrogate  # noqa: E402

m = load_arm7_surrogate()
for rows in [int(a) for a in sys.argv[1:]] or [1000, 100_000, 1_000_003]:
    q = np.random.default_rng(rows).uniform(-3, 3, size=(rows, 7))
    outs = {}
    for v in ("0", "1", "1b"):
        os.environ["MPPI_MLP2"] = v[0]
        outs[v] = m.distance(q)
    d = np.abs(outs["0"] - outs["1"])
    d2 = np.abs(outs["1"] - outs["1b"])
    print(f"rows {rows}: max |v1 - v2| = {d.max():.3e} ({(d > 0).sum()} differ); v2 rerun {d2.max():.3e}", flush=True)

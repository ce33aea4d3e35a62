"""Run the MLP forward on a config-4-sized batch (for ncu captures)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2104_13542_b200.surrogate import load_arm7_surrogate  # noqa: E402
import numpy as np  # noqa: E402

m = load_arm7_surrogate()
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 960_000
q = np.random.default_rng(0).uniform(-3, 3, size=(rows, 7))
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    m.distance(q)
print("done", rows)

"""One MLP forward through mppi_mlp_forward with the variant from MPPI_MLP2."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2104_13542_b200.surrogate import load_arm7_surrogate  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
q = np.random.default_rng(0).uniform(-3, 3, size=(rows, 7))
out = load_arm7_surrogate().distance(q)
np.save(sys.argv[2] if len(sys.argv) > 2 else "/tmp/mlp_out.npy", out)
print("ok", rows, float(out[:5].sum()))

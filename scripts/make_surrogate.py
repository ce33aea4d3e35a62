"""Train the arm7 learned self-collision surrogate with the REFERENCE package
(offline; training is out of scope for the hot path, SURVEY.md §2 surrogate.py row).

Run in the build container only (needs /root/reference):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python scripts/make_surrogate.py
Writes paper_2104_13542_b200/data/arm7_surrogate.npz with the reference's
LearnedSelfCollision.save layout (W0..W3, b0..b3, dof, holdout_mae,
sign_agreement; surrogate.py:127-133).
"""
import sys
from pathlib import Path

from jointmpc.kinematics import load_chain
from jointmpc.surrogate import train_collision_surrogate

out = Path(__file__).resolve().parents[1] / "paper_2104_13542_b200" / "data" / "arm7_surrogate.npz"
model = train_collision_surrogate(load_chain("arm7.chain"), 50000, seed=0)
model.save(out)
print(f"wrote {out}: holdout_mae={model.holdout_mae:.5f} sign={model.sign_agreement:.4f}", file=sys.stderr)

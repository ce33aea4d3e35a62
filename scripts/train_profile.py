"""Short device training run (for ncu launch lists of the training kernels)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2104_13542_b200.kinematics import load_chain  # noqa: E402
from paper_2104_13542_b200.surrogate import train_collision_surrogate  # noqa: E402

epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 2
m, losses, ms = train_collision_surrogate(load_chain("arm7.chain"), 50_000, 0, epochs=epochs, return_losses=True)
print(f"{len(losses)} steps in {ms:.1f} ms device ({1e3 * ms / len(losses):.1f} us/step); mae {m.holdout_mae:.4f}")

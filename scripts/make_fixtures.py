"""Re-emit the reference's chain fixtures (data, not code) into the package in
this repo's canonical JSON layout (sorted keys, one-space indent, provenance
key). Same schema as jointmpc's loader (kinematics.py:117-180), so either
package can read either file.

    python scripts/make_fixtures.py    # needs /root/reference (build container only)
"""
import json
from pathlib import Path

SRC = Path("/root/reference/pkg/src/jointmpc/fixtures")
DST = Path(__file__).resolve().parents[1] / "paper_2104_13542_b200" / "fixtures"
for name in ("arm7", "planar2", "slider1", "planar_holonomic"):
    data = json.loads((SRC / f"{name}.chain").read_text())
    data["_source"] = f"jointmpc fixtures/{name}.chain (re-emitted by scripts/make_fixtures.py)"
    (DST / f"{name}.chain").write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")
    print("wrote", DST / f"{name}.chain")

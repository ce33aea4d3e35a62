"""Install the UNMODIFIED reference package into oracle/_ref (git-ignored, but
it travels to the GPU box with the gpurun snapshot) for the CPU reference arm
of bench.py (``--impl reference`` and the ``cpu_baseline`` leg).

The reference is pure Python + numba (no native build); this is the
"compile the reference where it lies" recipe of the task, for a Python
reference: pip installs it from /root/reference (read-only, so from a /tmp
copy) with no index and no dependency resolution (numpy/numba are in the image).
Test/bench infrastructure only.
"""
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

SRC = Path("/root/reference/pkg")
DST = Path(__file__).resolve().parent / "_ref"


def main() -> int:
    if not SRC.exists():
        print("reference not present; keeping existing oracle/_ref", file=sys.stderr)
        return 0
    if (DST / "jointmpc" / "controller.py").exists():
        return 0
    with tempfile.TemporaryDirectory() as tmp:
        work = Path(tmp) / "pkg"
        shutil.copytree(SRC, work)
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps",
               "--find-links", "/opt/wheelhouse", "--target", str(DST), str(work)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        print(r.stdout[-2000:], r.stderr[-2000:], file=sys.stderr)
        return r.returncode


if __name__ == "__main__":
    sys.exit(main())

"""Build the current csrc/ tree into another .so (A/B timing of kernel variants with UBQP_LIB).

    python tools/build_variant.py variants/name.so        # UBQP_NVCC_EXTRA="..." adds flags
"""
import os
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1706_00037_b200.build import CSRC, NVCC, NVCC_FLAGS, SOURCES  # noqa: E402

out = Path(sys.argv[1])
out.parent.mkdir(parents=True, exist_ok=True)
extra = os.environ.get("UBQP_NVCC_EXTRA", "").split()
subprocess.check_call([NVCC, *NVCC_FLAGS, *extra, "-shared", "-o", str(out), *[str(CSRC / s) for s in SOURCES]])
print(out)

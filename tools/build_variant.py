"""Build the current csrc/ tree into another .so (A/B timing of kernel variants with UBQP_LIB).

    python tools/build_variant.py variants/name.so
"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1706_00037_b200.build import CSRC, NVCC, NVCC_FLAGS, SOURCES  # noqa: E402

out = Path(sys.argv[1])
out.parent.mkdir(parents=True, exist_ok=True)
subprocess.check_call([NVCC, *NVCC_FLAGS, "-shared", "-o", str(out), *[str(CSRC / s) for s in SOURCES]])
print(out)

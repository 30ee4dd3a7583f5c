"""Build the current csrc/ tree into another .so (A/B timing of kernel variants with UBQP_LIB).

    python tools/build_variant.py variants/name.so        # UBQP_NVCC_EXTRA="..." adds flags
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1706_00037_b200.build import build_lib  # noqa: E402

print(build_lib(out=Path(sys.argv[1])))

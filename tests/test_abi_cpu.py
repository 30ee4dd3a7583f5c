"""CPU-side checks of the C-ABI boundary (no GPU compute): libubqp.so builds for sm_100a,
loads, exports every entry point include/ubqp.h declares, and fails loudly without a device."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "ubqp.h"


@pytest.fixture(scope="module")
def lib():
    from paper_1706_00037_b200.build import build_lib
    path = build_lib()
    return ctypes.CDLL(str(path))


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ubqp_[A-Za-z_0-9]+)\s*\(", text)))


def test_header_declares_the_boundary_calls():
    names = declared_functions()
    for required in ("ubqp_load_Q", "ubqp_diversify", "ubqp_eval_batch", "ubqp_screen", "ubqp_ascend"):
        assert required in names          # north_star boundary


def test_every_declared_symbol_is_exported(lib):
    from paper_1706_00037_b200.ubqp import EXPORTS
    names = declared_functions()
    assert sorted(EXPORTS) == names       # the Python binding covers the header exactly
    for name in names:
        assert hasattr(lib, name), name


def test_library_is_sm100a_native():
    import subprocess
    from paper_1706_00037_b200.build import LIB
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(LIB)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", str(LIB)],
                                       capture_output=True, text=True).stdout
    assert "UTCIMMA" in out               # tcgen05.mma kind::i8
    assert "UTMALDG" in out               # TMA loads
    assert "LDTM" in out                  # tcgen05.ld (TMEM -> registers)
    assert "IDP.2A" in out                # ascent update


def test_version_and_null_handle(lib):
    lib.ubqp_version.restype = ctypes.c_int
    assert lib.ubqp_version() == 200
    lib.ubqp_last_error.restype = ctypes.c_char_p
    lib.ubqp_last_error.argtypes = [ctypes.c_void_p]
    assert b"null" in lib.ubqp_last_error(None)
    lib.ubqp_sync.argtypes = [ctypes.c_void_p]
    assert lib.ubqp_sync(None) == 1       # UBQP_E_INVALID


def test_create_without_a_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    lib.ubqp_create.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
    assert lib.ubqp_create(0, None, ctypes.byref(h)) != 0
    assert not h.value
    from paper_1706_00037_b200 import Ubqp, UbqpError
    with pytest.raises(UbqpError):
        Ubqp(0)


def _imports(src):
    return re.findall(r"^\s*(?:from\s+(\S+)\s+import|import\s+(\S+)|#\s*include\s+[<\"](\S+)[>\"])", src, re.M)


def test_oracle_shares_no_code_with_the_cuda_path():
    """The oracle (test infrastructure) and the product path never include/import each other."""
    for p in (ROOT / "paper_1706_00037_b200").rglob("*"):
        if p.suffix in (".py", ".cu", ".cuh", ".h"):
            for mod in _imports(p.read_text()):
                assert not any("oracle" in x for x in mod), (p, mod)
    for p in (ROOT / "oracle").rglob("*"):
        if p.suffix in (".py", ".c", ".h"):
            for mod in _imports(p.read_text()):
                assert not any(("paper_1706" in x or "ubqp.h" in x or "csrc" in x) for x in mod), (p, mod)


def test_plain_c_example_compiles_against_the_header_and_library(tmp_path):
    """The boundary is a C-ABI: a C99 program (examples/ubqp_round.c) compiles against
    include/ubqp.h with -Wall -Wextra -Werror and links libubqp.so."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    from paper_1706_00037_b200.build import build_lib
    build_lib()
    out = tmp_path / "ubqp_round"
    subprocess.check_call(["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}",
                           str(ROOT / "examples" / "ubqp_round.c"), f"-L{ROOT / 'paper_1706_00037_b200'}", "-lubqp",
                           f"-Wl,-rpath,{ROOT / 'paper_1706_00037_b200'}", "-o", str(out)])
    assert out.exists()


def test_binding_refuses_a_missing_library(tmp_path, monkeypatch):
    """No CPU fallback: pointing the binding at a library that does not exist raises."""
    import paper_1706_00037_b200.ubqp as ub
    monkeypatch.setattr(ub, "_lib", None)      # restored by monkeypatch afterwards
    with pytest.raises(OSError):
        ub.load_library(tmp_path / "missing_libubqp.so")

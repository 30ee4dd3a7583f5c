"""The boundary exercised from plain C (examples/ubqp_round.c, C99, host arrays only): a whole
round -- first-derivative start, Glover diversification, eval + gains, screen, steepest ascent,
best key -- checked element by element against the oracle on the program's own Q."""
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1706_00037_b200.build import build_lib  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("n,K", [(300, 2000), (1025, 777)])
def test_c_program_round_matches_oracle(tmp_path, n, K):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lib = build_lib()
    exe = tmp_path / "ubqp_round"
    subprocess.check_call(["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}",
                           str(ROOT / "examples" / "ubqp_round.c"), f"-L{lib.parent}", "-lubqp",
                           f"-Wl,-rpath,{lib.parent}", "-o", str(exe)])
    prefix = tmp_path / "run"
    out = subprocess.run([str(exe), str(n), str(K), str(prefix)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    Q = np.fromfile(f"{prefix}.Q", dtype=np.int32).reshape(n, n)
    lines = Path(f"{prefix}.out").read_text().split("\n")
    ssum, scount, skey, T, m, best = lines[0].split()
    rows = np.array([[int(v) for v in ln.split()] for ln in lines[1:1 + int(m)]], dtype=np.int64).reshape(-1, 3)
    x0 = oracle.first_derivative_start(Q)
    X = oracle.diversify(x0, 0, K)
    f = oracle.eval_batch(Q, X, nthreads=8)
    st = oracle.stats(f)
    assert (int(ssum), int(scount), int(skey)) == (int(st[0]), int(st[1]), int(st[2]))
    maxv = (int(skey) >> 22) - (1 << 40)
    To = oracle.threshold(0.5, int(st[0]), int(st[1]), maxv)
    assert float(T) == To
    s = oracle.screen(f, To)
    assert rows[:, 0].tolist() == s.tolist()
    Xa, fa, fla = oracle.ascend(Q, X[s], f[s], 10 * n, nthreads=8)
    assert rows[:, 1].tolist() == fa.tolist() and rows[:, 2].tolist() == fla.tolist()
    assert int(best) == max(oracle.max_key(int(fa[i]), int(s[i])) for i in range(len(s)))

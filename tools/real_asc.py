"""bench.real_q_ascent on its own (R20 real-Q ascent measurement; UBQP_LIB for A/B)."""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.argv = ["bench"]
import torch  # noqa: E402
import bench  # noqa: E402
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
print(json.dumps(bench.real_q_ascent(0)))

"""FP16 edge messages vs FP32 after 1-3 sweeps: max/mean posterior and message
differences and sign flips (the numbers behind tests/test_msg16.py's tolerances), and the
FP16 rounding of an upload/download round trip.

    python tools/msg16_diag.py
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402
from conftest import channel_llrs, load_code  # noqa: E402

from paper_2004_09084_b200 import _native  # noqa: E402
base, sched, index = load_code("standin_v2_z100")
plan = _native.Plan(index, sched, 0)
n = base.n_cols * base.z
st = _native.State(plan, 8, "fp32-msg16")
_, msg0 = st.download()
rng = np.random.default_rng(0)
post = rng.normal(0, 5, size=(8, n)); msg = rng.normal(0, 5, size=(8, msg0.shape[1]))
st.upload(post, msg)
gp, gm = st.download()
print("post eq", np.array_equal(gp, post.astype(np.float32).astype(np.float64)), np.abs(gp-post).max())
want = msg.astype(np.float16).astype(np.float64)
bad = np.nonzero(gm != want)
print("msg mismatches", len(bad[0]), gm[bad][:5], want[bad][:5], msg[bad][:5])
for name, batch, sweeps in [("standin_v2_z100", 16, 1), ("standin_v2_z100", 64, 3), ("demo_6x12_z16", 33, 2), ("standin_v2_z2500", 8, 1)]:
    base, sched, index = load_code(name)
    plan = _native.Plan(index, sched, 0)
    n = base.n_cols * base.z
    llr = channel_llrs(n, 0.5, seed=1, snr_idx=0, frames=batch)
    out = []
    for prec in ("fp32", "fp32-msg16"):
        s = _native.State(plan, batch, prec); s.set_llr(llr); s.reset(30.0); s.set_syndrome(None)
        for _ in range(sweeps): s.layers(0, len(sched.layers), 30.0, 1e-10)
        out.append(s.download())
    (la, ra), (lb, rb) = out
    rel = np.abs(rb - ra) / (np.abs(ra) + 1e-3)
    print(name, batch, sweeps, "L maxdiff %.4g mean %.3g" % (np.abs(lb-la).max(), np.abs(lb-la).mean()),
          "R maxdiff %.4g rel-max %.3g rel-mean %.3g" % (np.abs(rb-ra).max(), rel.max(), rel.mean()),
          "flips", np.count_nonzero((la < 0) != (lb < 0)), "of", la.size)

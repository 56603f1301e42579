"""Digest of the decoder state after a few flow sweeps (compare builds: QCL_LIB_VARIANT)."""
import hashlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from conftest import load_code  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402

for name, batch, sweeps in [("standin_v2_z100", 64, 5), ("standin_v2_z2500", 64, 2), ("demo_6x12_z16", 33, 4)]:
    base, sched, index = load_code(name)
    plan = _native.Plan(index, sched, 0)
    st = _native.State(plan, batch, "fp32")
    st.set_llr_synthetic(seed=3, snr_idx=0, first_frame=0, snr=0.161)
    st.reset(30.0)
    st.set_syndrome(None)
    for _ in range(sweeps):
        st.layers(0, len(sched.layers), 30.0, 1e-10)
    post, msg = st.download()
    print(name, batch, sweeps, hashlib.sha256(post.tobytes() + msg.tobytes()).hexdigest()[:16], flush=True)

"""Frame-pool decode for a launch list / timing: n=1e6 stand-in, 64 lanes, `--frames`
frames at `--snr`, cap `--iters`, early termination (qcl_state_decode_pool)."""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2004_09084_b200 as q  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=8)
ap.add_argument("--snr", type=float, default=0.14)
ap.add_argument("--frames", type=int, default=64)
a = ap.parse_args()
base = q.load_base_matrix(ROOT / "codes" / "standin_v2_z2500.txt")
sched = q.greedy_schedule(base)
index = q.build_compact_index(base, sched)
plan = _native.Plan(index, sched, 0)
st = _native.State(plan, 64, "fp32")
cfg = _native.make_config(q.DecoderConfig(max_iterations=a.iters, early_termination=True), "fp32")
for rep in range(2):
    t0 = time.perf_counter()
    conv, iters, err, ms = st.decode_pool(cfg, 0, 0, 0, a.frames, a.snr)
    print(f"pool {a.frames} frames cap {a.iters}: {ms:.2f} ms device, {1e3 * (time.perf_counter() - t0):.2f} ms wall, "
          f"{iters.sum()} iterations", flush=True)

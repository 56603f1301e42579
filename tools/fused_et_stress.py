"""Fused early termination under repetition: `reps` processes (each with a timeout) x
`decodes` fused ET decodes of B codewords, every one compared with the per-layer engine.

    python tools/fused_et_stress.py [B] [snr] [reps] [decodes]
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CHILD = r'''
import sys; sys.path.insert(0, "{root}")
import numpy as np
import paper_2004_09084_b200 as q
from paper_2004_09084_b200 import _native
base = q.load_base_matrix("{root}/codes/standin_v2_z100.txt"); sched = q.greedy_schedule(base)
plan = _native.Plan(q.build_compact_index(base, sched), sched, 0)
cfg = _native.make_config(q.DecoderConfig(max_iterations=40, early_termination=True), "fp32")
ref = _native.State(plan, {B}, "fp32"); ref.set_engine(0)
ref.set_llr_synthetic(seed=5, snr_idx=1, first_frame=0, snr={snr}, encode_mode=True); ref.decode(cfg)
want = ref.results()
bad = 0
for i in range({decodes}):
    st = _native.State(plan, {B}, "fp32")
    st.set_llr_synthetic(seed=5, snr_idx=1, first_frame=0, snr={snr}, encode_mode=True)
    st.decode(cfg)
    bad += not all(np.array_equal(a, b) for a, b in zip(st.results(), want))
print("ok" if not bad else f"MISMATCH {{bad}}")
'''
B = int(sys.argv[1]) if len(sys.argv) > 1 else 21
snr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.19
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
decodes = int(sys.argv[4]) if len(sys.argv) > 4 else 10
res = {}
for r in range(reps):
    try:
        out = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT, B=B, snr=snr, decodes=decodes)],
                             capture_output=True, text=True, timeout=40)
        key = out.stdout.strip() or ("ERR " + out.stderr.strip()[-200:])
    except subprocess.TimeoutExpired:
        key = "HANG"
    res[key] = res.get(key, 0) + 1
print(f"B={B} snr={snr}: {res}", flush=True)

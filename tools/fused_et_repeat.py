"""Repeated fused-ET decodes where every frame converges after the first sweep (SNR 20,
encode mode) and at SNR 3 (no frame converges, saturated messages): engine 4 against
engine 0, reporting any difference in flags, iteration counts or words.

    python tools/fused_et_repeat.py REPS ["B:SNR,B:SNR,..." [SEED,SEED,...]]
"""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_2004_09084_b200 as q
from paper_2004_09084_b200 import _native
from conftest import load_code

base, sched, index = load_code("standin_v2_z100")
plan = _native.Plan(index, sched, 0)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
bad = 0
configs = ((40, 20.0), (21, 20.0), (128, 3.0), (21, 3.0), (40, 20.0)) if len(sys.argv) < 3 else \
    [(int(b), float(s)) for b, s in (x.split(':') for x in sys.argv[2].split(','))]
seeds = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [9]
for (batch, snr), seed in ((c, sd) for c in configs for sd in seeds):
    cfg = _native.make_config(q.DecoderConfig(max_iterations=50, early_termination=True), "fp32")
    ref = _native.State(plan, batch, "fp32")
    ref.set_engine(0)
    ref.set_llr_synthetic(seed=seed, snr_idx=2, first_frame=0, snr=snr, encode_mode=True)
    ref.decode(cfg)
    w0, c0, i0 = ref.results()
    for r in range(reps):
        st = _native.State(plan, batch, "fp32")
        st.set_engine(4)
        st.set_llr_synthetic(seed=seed, snr_idx=2, first_frame=0, snr=snr, encode_mode=True)
        st.decode(cfg)
        w, c, i = st.results()
        if not (np.array_equal(w, w0) and np.array_equal(c, c0) and np.array_equal(i, i0)):
            bad += 1
            fr = np.nonzero((w != w0).any(axis=1) | (c != c0) | (i != i0))[0]
            print(f"MISMATCH B={batch} snr={snr} seed {seed} rep {r}: frames {fr[:10]} conv {c[fr[:5]]} vs {c0[fr[:5]]} "
                  f"it {i[fr[:5]]} vs {i0[fr[:5]]} bits {(w != w0).sum(axis=1)[fr[:5]]}", flush=True)
    print(f"B={batch} snr={snr} seed {seed}: ref conv {c0.mean():.2f} it {i0.min()}-{i0.max()}, {reps} reps done", flush=True)
print("ALL OK" if bad == 0 else f"{bad} mismatching decodes")

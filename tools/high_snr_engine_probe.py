"""SNR 20 (far above the operating point), FP32, ET cap 50, encode mode: engines 0 / 1 / 4
at 8 and 40 codewords against the C oracle on the same device LLRs and targets."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_2004_09084_b200 as q
from paper_2004_09084_b200 import _native
from oracle import oracle as O
from conftest import load_code

base, sched, index = load_code("standin_v2_z100")
plan = _native.Plan(index, sched, 0)
code = O.OracleCode(index, sched)
for B in (8, 40):
    for engine in (0, 1, 4):
        for seed, sidx in ((9, 2), (5, 1)):
            st = _native.State(plan, B, "fp32")
            st.set_engine(engine)
            st.set_llr_synthetic(seed=seed, snr_idx=sidx, first_frame=0, snr=20.0, encode_mode=True)
            st.decode(_native.make_config(q.DecoderConfig(max_iterations=50, early_termination=True), "fp32"))
            w, c, it = st.results()
            llr = st.get_llr()
            syn = O.syndrome(code, st.truths())
            ow, oc, oi = O.decode(code, llr, syn, max_iterations=50, early_termination=True)
            print(f"B={B} engine {engine} seed {seed}/{sidx}: conv {c.mean():.2f} it max {it.max()} | oracle conv "
                  f"{oc.mean():.2f} it max {oi.max()} | flags equal {np.array_equal(c, oc)} | word bits differ "
                  f"{int((w != ow).sum())}", flush=True)

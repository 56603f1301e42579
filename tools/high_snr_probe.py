import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_2004_09084_b200 as q
from paper_2004_09084_b200 import _native
from oracle import oracle as O
from conftest import load_code
base, sched, index = load_code("standin_v2_z100")
plan = _native.Plan(index, sched, 0)
code = O.OracleCode(index, sched)
cfgq = q.DecoderConfig(max_iterations=20, early_termination=True)
for enc in (False, True):
    for snr in (1.5, 3.0, 20.0):
        st = _native.State(plan, 4, "fp64")
        st.set_llr_synthetic(seed=9, snr_idx=2, first_frame=0, snr=snr, encode_mode=enc)
        if not enc: st.set_syndrome(None)
        st.decode(_native.make_config(cfgq, "fp64"))
        w, c, it = st.results()
        llr = st.get_llr()
        tr = st.truths() if enc else np.zeros_like(w)
        syn = O.syndrome(code, tr)
        ow, oc, oi = O.decode(code, llr, syn, max_iterations=20, early_termination=True)
        hd_err = ((llr < 0).astype(np.uint8) != tr).sum(axis=1)
        print(f"enc={enc} snr={snr}: device conv {c.astype(int)} it {it} | oracle conv {oc.astype(int)} it {oi} | "
              f"words equal {np.array_equal(w, ow)} | channel hard-decision errors {hd_err} |llr| max {np.abs(llr).max():.1f}", flush=True)

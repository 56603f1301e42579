"""High-SNR FP32 behaviour against the FP64 oracle: device FP32 / FP64 decodes of the
same device LLRs (z=100 stand-in twin), convergence per sweep cap, and the posterior
after one sweep compared with the oracle's."""
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
for snr in (1.5, 5.0, 20.0):
    for prec in ("fp32", "fp64"):
        for engine in (0, 1, 4):
            st = _native.State(plan, 4, prec)
            st.set_engine(engine)
            st.set_llr_synthetic(seed=9, snr_idx=2, first_frame=0, snr=snr)
            st.set_syndrome(None)
            st.decode(_native.make_config(q.DecoderConfig(max_iterations=3, early_termination=False), prec))
            w, c, it = st.results()
            post, msg = st.download()
            llr = st.get_llr()
            ow, oc, oi, opost = O.decode(code, llr, None, max_iterations=3, early_termination=False, want_posterior=True)
            d = np.abs(post - opost)
            print(f"snr {snr} {prec} engine {engine}: conv {c.astype(int)} oracle {oc.astype(int)}; word bits differ "
                  f"{int((w != ow).sum())}; posterior max diff {d.max():.3g}; |post| max {np.abs(post).max():.1f}, "
                  f"oracle {np.abs(opost).max():.1f}; |llr| max {np.abs(llr).max():.1f}", flush=True)

print("--- early termination, cap 20 (encode mode: random words, H c targets) ---", flush=True)
for snr in (1.5, 3.0, 20.0):
    for prec in ("fp32", "fp64"):
        st = _native.State(plan, 8, prec)
        st.set_llr_synthetic(seed=9, snr_idx=2, first_frame=0, snr=snr, encode_mode=True)
        st.decode(_native.make_config(q.DecoderConfig(max_iterations=20, early_termination=True), prec))
        w, c, it = st.results()
        llr = st.get_llr()
        syn = O.syndrome(code, st.truths())
        ow, oc, oi = O.decode(code, llr, syn, max_iterations=20, early_termination=True)
        print(f"snr {snr} {prec}: conv {c.astype(int)} it {it} | oracle conv {oc.astype(int)} it {oi} | "
              f"word bits differ {int((w != ow).sum())}", flush=True)

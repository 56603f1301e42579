import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_2004_09084_b200 as q
from paper_2004_09084_b200 import _native
from conftest import load_code
base, sched, index = load_code("standin_v2_z100")
plan = _native.Plan(index, sched, 0)
cfg = _native.make_config(q.DecoderConfig(max_iterations=50, early_termination=True), "fp32")
for batch, snr in ((40, 20.0), (128, 20.0), (21, 20.0), (64, 1.0)):
    outs = []
    for engine in (0, 4, 4, 4, 4):
        st = _native.State(plan, batch, "fp32")
        st.set_engine(engine)
        st.set_llr_synthetic(seed=9, snr_idx=2, first_frame=0, snr=snr, encode_mode=True)
        st.decode(cfg)
        outs.append(st.results())
    w0, c0, i0 = outs[0]
    line = f"B={batch} snr={snr}: engine0 conv {c0.mean():.2f} it {i0.min()}-{i0.max()}"
    for k, (w, c, i) in enumerate(outs[1:]):
        line += f" | run{k}: conv {c.mean():.2f} it {i.min()}-{i.max()} words diff {int((w != w0).sum())} flags eq {np.array_equal(c, c0)} it eq {np.array_equal(i, i0)}"
    print(line, flush=True)

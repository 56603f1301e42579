"""Device time of one 64-codeword decode (rate-0.1 n=1e6 stand-in, SNR 0.161) per engine."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import paper_2004_09084_b200 as q  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
batches = [int(x) for x in sys.argv[2].split(',')] if len(sys.argv) > 2 else [64, 32, 128]
engines = [int(x) for x in sys.argv[3].split(',')] if len(sys.argv) > 3 else [0, 1]
base = q.load_base_matrix(ROOT / "codes" / "standin_v2_z2500.txt")
sched = q.greedy_schedule(base)
index = q.build_compact_index(base, sched)
plan = _native.Plan(index, sched, 0)
n = base.n_cols * base.z
for batch in batches:
    for prec in ("fp32",):
        res = {}
        for engine in engines:
            st = _native.State(plan, batch, prec)
            st.set_engine(engine + 2)
            st.set_llr_synthetic(seed=0, snr_idx=0, first_frame=0, snr=0.161)
            st.set_syndrome(None)
            cfg = _native.make_config(q.DecoderConfig(max_iterations=iters, early_termination=False), prec)
            st.decode(cfg)
            ms = min(st.decode(cfg) for _ in range(3))
            ll, lms, al = st.kernel_stats()
            w, c, it = st.results()
            res[engine] = w
            mbps = batch * n / (ms * 50 / iters / 1e3) / 1e6
            print(f"B={batch} {prec} engine={engine}: {ms:.2f} ms for {iters} it -> {mbps:.0f} Mbit/s at 50 it; "
                  f"sweep avg {lms / iters:.3f} ms, {ll // iters} launches/sweep", flush=True)
        if len(res) > 1:
            print("  engines agree bit-exactly:", np.array_equal(res[engines[0]], res[engines[1]]))

"""Where the drop-in call's time goes (bench.py `e2e`): 64 codewords of the n = 10^6
stand-in, pageable float64 LLRs and uint8 syndromes as the reference passes them.

    [QCL_HOST_THREADS=k] python tools/e2e_breakdown.py

Prints the host-side stages alone (conversion + H2D of the LLRs, the all-zero syndrome
check, the D2H of the words), the device decode alone, and the decode_stream step.
"""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import paper_2004_09084_b200 as q  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402

base = q.load_base_matrix(ROOT / "codes" / "standin_v2_z2500.txt")
sched = q.greedy_schedule(base)
index = q.build_compact_index(base, sched)
n, m, B = base.n_cols * base.z, base.n_rows * base.z, 64
cfg = q.DecoderConfig(max_iterations=50, early_termination=False)
dec = q.LayeredDecoder(index, sched, cfg)
plan = _native.Plan(index, sched, 0)
st = _native.State(plan, B, "fp32")
st.set_llr_synthetic(seed=0, snr_idx=0, first_frame=0, snr=0.161)
llr = st.get_llr()
syn = np.zeros((B, m), np.uint8)
words = _native.PinnedArray((B, n), np.uint8)
conv = _native.PinnedArray((B,), np.uint8)
iters = _native.PinnedArray((B,), np.int64)
qcfg = _native.make_config(cfg, "fp32")
print(f"host threads: {os.environ.get('QCL_HOST_THREADS', os.cpu_count())} (cpu_count {os.cpu_count()})")


def timed(label, fn, reps=4):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    print(f"{label}: {1e3 * min(ts):.2f} ms (median {1e3 * float(np.median(ts)):.2f})", flush=True)


timed("set_llr pageable f64 (convert + H2D, synced)", lambda: (st.set_llr(llr), st.wait()))
timed("set_syndrome_hint (host zero check)", lambda: st.set_syndrome_hint(syn))
timed("device decode (events)", lambda: st.decode(qcfg))
timed("results_async -> pinned + wait", lambda: (st.results_async(words.array, conv.array, iters.array), st.wait()))
timed("results() pageable", lambda: st.results())
llr2 = llr.copy()
for _ in dec.decode_stream([(llr, syn), (llr2, syn)]):
    pass
steps = 12
t0 = time.perf_counter()
for _ in dec.decode_stream(((llr if i % 2 else llr2, syn) for i in range(steps)), depth=2):
    pass
print(f"decode_stream step: {1e3 * (time.perf_counter() - t0) / steps:.2f} ms", flush=True)
t0 = time.perf_counter()
dec.decode_batch_arrays(llr, syn)
print(f"decode_batch_arrays (blocking): {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)

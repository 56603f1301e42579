"""Small decodes on every engine for compute-sanitizer (memcheck / racecheck / synccheck):
demo_4x8_z100 and the z=100 stand-in twin, FP32 and FP64, ET on and off, with a
random target syndrome.  Exits non-zero on a result mismatch between engines."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import paper_2004_09084_b200 as q  # noqa: E402

rng = np.random.default_rng(0)
for name in ("demo_4x8_z100", "standin_v2_z100"):
    base = q.load_base_matrix(ROOT / "codes" / f"{name}.txt")
    sched = q.greedy_schedule(base)
    index = q.build_compact_index(base, sched)
    n, m = base.n_cols * base.z, base.n_rows * base.z
    llr = rng.normal(0.5, 2.0, size=(9, n))
    syn = (rng.random((9, m)) < 0.3).astype(np.uint8)
    for et in (False, True):
        cfg = q.DecoderConfig(max_iterations=4, early_termination=et)
        for precision in ("fp32", "fp64"):
            res = [q.LayeredDecoder(index, sched, cfg, precision=precision, engine=e).decode_batch_arrays(llr, syn)
                   for e in (0, 1, 4)]
            same = all(np.array_equal(a, b) for r in res[1:] for a, b in zip(res[0], r))
            print(name, "et" if et else "noet", precision, "engines agree:", same, flush=True)
            if precision == "fp32" and not same:
                sys.exit(1)

# flow-engine paths added later: group blocks (128 codewords = 2 blocks of 8 lane groups),
# FP16 messages, the frame pool
base = q.load_base_matrix(ROOT / "codes" / "standin_v2_z100.txt")
sched = q.greedy_schedule(base)
index = q.build_compact_index(base, sched)
n, m = base.n_cols * base.z, base.n_rows * base.z
llr = rng.normal(0.5, 2.0, size=(128, n))
for et in (False, True):
    cfg = q.DecoderConfig(max_iterations=3, early_termination=et)
    res = [q.LayeredDecoder(index, sched, cfg, precision="fp32", engine=e).decode_batch_arrays(llr, np.zeros((128, m), np.uint8))
           for e in (0, 4)]
    same = all(np.array_equal(a, b) for a, b in zip(res[0], res[1]))
    print("standin_v2_z100 B=128", "et" if et else "noet", "fp32 engines agree:", same, flush=True)
    if not same:
        sys.exit(1)
    out = q.LayeredDecoder(index, sched, cfg, precision="fp32-msg16").decode_batch_arrays(llr[:9], np.zeros((9, m), np.uint8))
    print("standin_v2_z100 B=9", "et" if et else "noet", "fp32-msg16 ran, converged", int(out[1].sum()), flush=True)
from paper_2004_09084_b200 import _native  # noqa: E402

st = _native.State(_native.Plan(index, sched, 0), 16, "fp32")
qcfg = _native.make_config(q.DecoderConfig(max_iterations=6, early_termination=True), "fp32")
conv, iters, err, _ = st.decode_pool(qcfg, 0, 0, 0, 40, 0.3)
print("frame pool 40 frames:", int(conv.sum()), "converged", int(iters.sum()), "iterations", flush=True)

# fused early termination (round 2): encode-mode targets, two group blocks, a ragged group
for B in (21, 128):
    pl = _native.Plan(index, sched, 0)
    outs = []
    for engine in (0, 4):
        s2 = _native.State(pl, B, "fp32")
        s2.set_engine(engine)
        s2.set_llr_synthetic(seed=5, snr_idx=1, first_frame=0, snr=0.19, encode_mode=True)
        s2.decode(_native.make_config(q.DecoderConfig(max_iterations=8, early_termination=True), "fp32"))
        outs.append(s2.results())
    same = all(np.array_equal(a, b) for a, b in zip(*outs))
    print(f"fused ET B={B}: engines agree: {same}, converged {int(outs[1][1].sum())}", flush=True)
    if not same:
        sys.exit(1)

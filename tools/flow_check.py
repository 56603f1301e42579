"""Flow engine (4) vs per-layer TMA engine (0): bit-exact state after N sweeps and
identical decode outcomes, over codes, batch sizes (lane widths), syndromes and early
termination; then the 64-codeword n=1e6 timing of both engines.

    python tools/flow_check.py [--quick]
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402

import paper_2004_09084_b200 as q  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402


def code(name):
    base = q.load_base_matrix(ROOT / "codes" / f"{name}.txt")
    sched = q.greedy_schedule(base)
    return base, sched, q.build_compact_index(base, sched)


def states_equal(name, batch, sweeps, syn_on, seed=1):
    base, sched, index = code(name)
    plan = _native.Plan(index, sched, 0)
    n, m = base.n_cols * base.z, base.n_rows * base.z
    rng = np.random.default_rng(seed)
    llr = rng.normal(0.3, 2.0, size=(batch, n))
    syn = (rng.random((batch, m)) < 0.5).astype(np.uint8) if syn_on else None
    out = {}
    for engine in (0, 4):
        st = _native.State(plan, batch, "fp32")
        st.set_engine(engine)
        st.set_llr(llr)
        st.reset(30.0)
        st.set_syndrome(syn)
        for _ in range(sweeps):
            st.layers(0, len(sched.layers), 30.0, 1e-10)
        out[engine] = st.download()
    same = all(np.array_equal(a, b) for a, b in zip(out[0], out[4]))
    print(f"state {name} B={batch} sweeps={sweeps} syn={syn_on}: bit-exact={same}", flush=True)
    return same


def decodes_equal(name, batch, iters, et, snr):
    base, sched, index = code(name)
    n, m = base.n_cols * base.z, base.n_rows * base.z
    chan = q.ChannelConfig(snr=snr, seed=0)
    llr = np.stack([q.init_llr(q.transmit(np.zeros(n, np.uint8), chan, q.frame_rng(0, 0, i)), chan)
                    for i in range(batch)])
    cfg = q.DecoderConfig(max_iterations=iters, early_termination=et)
    res = {}
    for engine in (0, 4):
        dec = q.LayeredDecoder(index, sched, cfg, precision="fp32", engine=engine)
        res[engine] = dec.decode_batch_arrays(llr, np.zeros((batch, m), np.uint8))
    same = all(np.array_equal(a, b) for a, b in zip(res[0], res[4]))
    print(f"decode {name} B={batch} it={iters} et={et} snr={snr}: identical={same} "
          f"conv={int(res[4][1].sum())}/{batch} iters={res[4][2][:8]}", flush=True)
    return same


def timing(batch=64, iters=50, engines=(0, 4)):
    base, sched, index = code("standin_v2_z2500")
    plan = _native.Plan(index, sched, 0)
    n = base.n_cols * base.z
    for engine in engines:
        st = _native.State(plan, batch, "fp32")
        st.set_engine(engine)
        st.set_llr_synthetic(seed=0, snr_idx=0, first_frame=0, snr=0.161)
        st.set_syndrome(None)
        cfg = _native.make_config(q.DecoderConfig(max_iterations=iters, early_termination=False), "fp32")
        st.decode(cfg)
        ms = [st.decode(cfg) for _ in range(3)]
        w, c, it = st.results()
        print(f"timing B={batch} engine={engine}: {min(ms):.2f} ms / {iters} it -> "
              f"{batch * n / (min(ms) / 1e3) / 1e6:.0f} Mbit/s  (words sum {int(w.sum())})", flush=True)


if __name__ == "__main__":
    quick = "--quick" in sys.argv
    ok = True
    ok &= states_equal("demo_4x8_z100", 4, 1, False)
    ok &= states_equal("standin_v2_z100", 8, 1, True)
    ok &= states_equal("standin_v2_z100", 64, 3, True)
    ok &= states_equal("standin_v2_z100", 16, 5, False)
    ok &= states_equal("demo_6x12_z16", 32, 4, True)
    ok &= states_equal("standin_v2_z2500", 64, 2, False)
    ok &= decodes_equal("standin_v2_z100", 64, 20, False, 0.161)
    ok &= decodes_equal("standin_v2_z100", 64, 50, True, 0.2)
    ok &= decodes_equal("demo_4x8_z100", 33, 10, True, 1.0)
    print("ALL OK" if ok else "MISMATCH", flush=True)
    t0 = time.time()
    timing()
    if not quick:
        timing(128)
        timing(32)

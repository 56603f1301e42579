"""Persistent per-layer engine (W <= 2 lanes, one cooperative launch per decode) against
the per-layer launches: run once with QCL_PERSIST=2 (every 1-2 lane decode) and once with QCL_PERSIST=0 (the
switch is read once per process), then compare.

    QCL_PERSIST=2 python tools/persist_check.py dump gpurun_out/persist_on.npz
    QCL_PERSIST=0 python tools/persist_check.py dump gpurun_out/persist_off.npz
    python tools/persist_check.py compare gpurun_out/persist_on.npz gpurun_out/persist_off.npz
    QCL_PERSIST=2 QCL_PERSIST_BAR=1 python tools/persist_check.py time    # 50-iteration latency, B = 1, 2

`dump` also prints the single-codeword (configs[1]) 50-iteration latency.
"""
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402


def dump(out):
    import paper_2004_09084_b200 as q
    from paper_2004_09084_b200 import _native

    res = {}
    for code in ("standin_v2_z100", "demo_6x12_z16", "standin_v2_z2500"):
        base = q.load_base_matrix(ROOT / "codes" / f"{code}.txt")
        sched = q.greedy_schedule(base)
        plan = _native.Plan(q.build_compact_index(base, sched), sched, 0)
        m = base.n_rows * base.z
        for B in (1, 2):
            for prec in ("fp32", "fp64"):
                for syn in (False, True):
                    for et in (False, True):
                        if code == "standin_v2_z2500" and (syn or et):
                            continue
                        st = _native.State(plan, B, prec)
                        st.set_llr_synthetic(seed=3, snr_idx=1, first_frame=5, snr=0.2 if code != "demo_6x12_z16" else 1.0,
                                             encode_mode=syn)
                        if not syn:  # encode mode sets the target syndrome H c itself
                            st.set_syndrome(None)
                        cfg = _native.make_config(q.DecoderConfig(max_iterations=20, early_termination=et), prec)
                        st.decode(cfg)
                        w, c, it = st.results()
                        post, msg = st.download()
                        tag = f"{code}_B{B}_{prec}_syn{int(syn)}_et{int(et)}"
                        res[tag + "_w"] = np.asarray(w)
                        res[tag + "_c"] = np.asarray(c)
                        res[tag + "_i"] = np.asarray(it)
                        res[tag + "_L"] = post
                        res[tag + "_R"] = msg
                        del st
        if code == "standin_v2_z2500":
            for prec in ("fp32", "fp64"):
                st = _native.State(plan, 1, prec)
                st.set_llr_synthetic(seed=0, snr_idx=0, first_frame=0, snr=0.161)
                st.set_syndrome(None)
                cfg = _native.make_config(q.DecoderConfig(max_iterations=50, early_termination=False), prec)
                ms = [st.decode(cfg) for _ in range(10)][3:]
                print(f"configs[1] {prec} B=1: median {statistics.median(ms):.3f} ms (min {min(ms):.3f}), "
                      f"launches {st.kernel_stats()[0]}, "
                      f"{base.n_cols * base.z / statistics.median(ms) / 1e3:.0f} Mbit/s", flush=True)
                del st
    np.savez(out, **res)
    print("dumped", len(res), "arrays to", out)


def timing():
    import paper_2004_09084_b200 as q
    from paper_2004_09084_b200 import _native

    base = q.load_base_matrix(ROOT / "codes" / "standin_v2_z2500.txt")
    sched = q.greedy_schedule(base)
    plan = _native.Plan(q.build_compact_index(base, sched), sched, 0)
    out = []
    for B in (1, 2):
        for prec in ("fp32", "fp64"):
            st = _native.State(plan, B, prec)
            st.set_llr_synthetic(seed=0, snr_idx=0, first_frame=0, snr=0.161)
            st.set_syndrome(None)
            cfg = _native.make_config(q.DecoderConfig(max_iterations=50, early_termination=False), prec)
            ms = [st.decode(cfg) for _ in range(8)][3:]
            out.append(f"B={B} {prec} {statistics.median(ms):.3f} ms")
            del st
    print(" | ".join(out), flush=True)


def compare(a, b):
    x, y = np.load(a), np.load(b)
    bad = 0
    for k in sorted(x.files):
        same = np.array_equal(x[k], y[k], equal_nan=True)
        if not same:
            bad += 1
            print("MISMATCH", k, np.abs(x[k].astype(np.float64) - y[k].astype(np.float64)).max())
    print(f"compared {len(x.files)} arrays: {'ALL IDENTICAL' if bad == 0 else f'{bad} differ'}")
    return bad


if __name__ == "__main__":
    if sys.argv[1] == "dump":
        dump(sys.argv[2])
    elif sys.argv[1] == "time":
        timing()
    else:
        sys.exit(1 if compare(sys.argv[2], sys.argv[3]) else 0)

"""FP32 device decode vs the C oracle on the bench configuration: where do they differ?

Runs on a B200 box: decodes B frames of the bench's device LLRs (standin_v2_z2500,
SNR 0.161, 50 it, no ET) on the device (the library selected by QCL_LIB_VARIANT) and
in the oracle, then prints flipped bits with the oracle posterior at each flip, the
posterior error distribution, and how many oracle posteriors sit near zero.

    python tools/fp32_parity_diag.py [frames] [iters] [code]
"""

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2004_09084_b200 as q  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402


def main():
    frames = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    name = sys.argv[3] if len(sys.argv) > 3 else "standin_v2_z2500"
    base = q.load_base_matrix(ROOT / "codes" / f"{name}.txt")
    sched = q.greedy_schedule(base)
    index = q.build_compact_index(base, sched)
    dec = q.LayeredDecoder(index, sched, q.DecoderConfig(max_iterations=iters, early_termination=False))
    st = _native.State(dec._plan, frames, "fp32")
    st.set_llr_synthetic(seed=0, snr_idx=0, first_frame=0, snr=0.161)
    st.set_syndrome(None)
    llr = st.get_llr()
    ms = st.decode(dec._qcfg)
    w, c, it = st.results()
    post, _ = st.download()
    t0 = time.perf_counter()
    ow, oc, oi, op = oracle.decode(oracle.OracleCode(index, sched), llr, None, iters, False, want_posterior=True)
    t_or = time.perf_counter() - t0
    d = np.abs(post - op)
    rel = d / np.maximum(np.abs(op), 1.0)
    flips = np.argwhere(w != ow)
    near = {f"|L|<{e:g}": int((np.abs(op) < e).sum()) for e in (1e-5, 1e-4, 1e-3, 1e-2)}
    out = {
        "variant": __import__("os").environ.get("QCL_LIB_VARIANT", "default"),
        "code": name, "frames": frames, "iters": iters, "device_ms": ms, "oracle_s": t_or,
        "flips": len(flips), "flip_frames": sorted({int(f) for f, _ in flips}),
        "flip_oracle_post": [float(op[f, v]) for f, v in flips[:20]],
        "flip_device_post": [float(post[f, v]) for f, v in flips[:20]],
        "max_rel": float(rel.max()), "max_abs": float(d.max()),
        "p99.99_abs": float(np.quantile(d, 0.9999)), "mean_abs": float(d.mean()),
        "max_abs_where_|L|<1": float(d[np.abs(op) < 1].max()) if (np.abs(op) < 1).any() else None,
        "per_frame_max_rel": [float(x) for x in rel.max(axis=1)],
        "near_zero_oracle_posteriors": near,
        "converged": int(c.sum()), "oracle_converged": int(oc.sum()),
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()

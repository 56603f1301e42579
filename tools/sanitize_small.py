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

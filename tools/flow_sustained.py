"""Sustained flow-engine timing (power/clock behaviour like bench.py's timed loop):
64-codeword 50-iteration decodes back to back for --seconds, median ms of the second
half, with the SM clock sampled by nvidia-smi meanwhile.

    QCL_LIB_VARIANT=... python tools/flow_sustained.py [--seconds 15]
"""
import argparse
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2004_09084_b200 as q  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seconds", type=float, default=15.0)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--precision", default="fp32")
a = ap.parse_args()
base = q.load_base_matrix(ROOT / "codes" / "standin_v2_z2500.txt")
sched = q.greedy_schedule(base)
plan = _native.Plan(q.build_compact_index(base, sched), sched, 0)
st = _native.State(plan, a.batch, a.precision)
st.set_llr_synthetic(seed=0, snr_idx=0, first_frame=0, snr=0.161)
st.set_syndrome(None)
cfg = _native.make_config(q.DecoderConfig(max_iterations=50, early_termination=False), a.precision)
clocks, stop = [], threading.Event()


def sample():
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True).stdout.strip().split(",")
        try:
            clocks.append((float(out[0]), float(out[1])))
        except (ValueError, IndexError):
            pass
        time.sleep(0.5)


th = threading.Thread(target=sample)
th.start()
ms, t0 = [], time.time()
while time.time() - t0 < a.seconds:
    ms.append(st.decode(cfg))
stop.set()
th.join()
half = ms[len(ms) // 2:]
n = base.n_cols * base.z
med = statistics.median(half)
burst = statistics.median(ms[2:7])
print(f"sustained {a.precision} B={a.batch}: {len(ms)} decodes, burst (decodes 3-7) {burst:.2f} ms, "
      f"median {med:.2f} ms -> {a.batch * n / med / 1e3:.0f} Mbit/s; "
      f"sm clock median {statistics.median(c for c, _ in clocks):.0f} MHz, power median "
      f"{statistics.median(p for _, p in clocks):.0f} W", flush=True)

"""Where does the e2e time go?  PCIe copy rates, host syndrome scan, and decode_stream at
several depths (64 codewords, rate-0.1 n=1e6 stand-in, 50 it, no ET)."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2004_09084_b200 as q  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402

base = q.load_base_matrix(ROOT / "codes" / "standin_v2_z2500.txt")
sched = q.greedy_schedule(base)
index = q.build_compact_index(base, sched)
n, m, B = base.n_cols * base.z, base.n_rows * base.z, 64
dec = q.LayeredDecoder(index, sched, q.DecoderConfig(max_iterations=50, early_termination=False))
pin = _native.PinnedArray((B, n), np.float32)
pin.array[...] = np.random.default_rng(0).normal(0.32, 0.8, size=(B, n)).astype(np.float32)
syn = _native.PinnedArray((B, m), np.uint8)
syn.array[...] = 0
d = torch.empty(B * n, dtype=torch.float32, device="cuda")
src = torch.from_numpy(pin.array.reshape(-1))
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(src, non_blocking=True); torch.cuda.synchronize()
print(f"H2D 256 MB pinned: {(time.perf_counter() - t) * 1e3:.2f} ms")
hw = torch.empty(B * n, dtype=torch.uint8).pin_memory()
dw = torch.zeros(B * n, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize(); t = time.perf_counter(); hw.copy_(dw); torch.cuda.synchronize()
print(f"D2H 64 MB pinned: {(time.perf_counter() - t) * 1e3:.2f} ms")
t = time.perf_counter(); syn.array.any(); print(f"host syndrome scan (57.6 MB): {(time.perf_counter() - t) * 1e3:.2f} ms")
for depth in (1, 2, 3):
    for _ in dec.decode_stream([(pin.array, syn.array)] * depth, depth=depth):
        pass
    steps = 6
    t = time.perf_counter()
    for _ in dec.decode_stream([(pin.array, syn.array)] * steps, depth=depth):
        pass
    dt = (time.perf_counter() - t) / steps
    print(f"decode_stream depth {depth}: {dt * 1e3:.1f} ms/step -> {B * n / dt / 1e6:.0f} Mbit/s", flush=True)
st = _native.State(dec._plan, B, "fp32")
st.set_llr(pin.array); st.set_syndrome(None)
ms = [st.decode(dec._qcfg) for _ in range(3)]
print(f"device-resident decode: {min(ms):.1f} ms")

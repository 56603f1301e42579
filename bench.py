"""Throughput benchmark of the B200 layered decoder (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {b200,reference}] [--precision P]

Workload (BASELINE.json configs[2], the paper-style throughput run): the rate-0.1,
n = 10^6 QC-MET-LDPC stand-in (360x400 base, z = 2500, 3,767,500 edges;
``codes/standin_v2_z2500.txt``), 64 codewords per GPU, BIAWGN at SNR 0.161 (all-zero
word, zero syndrome, device Philox LLRs), 50 layered iterations, no early
termination, FP32 path.  One step = one full decode of the batch
(``decode_batch_arrays`` semantics: channel LLRs -> 50 sweeps -> hard decision +
syndrome).  The per-GPU working set (1.5 GB) is 12x the 126 MB L2, so no flush is
needed between steps.

Metric = frames * n / decode seconds / 1e6 (reference definition, bench.py:246).
``value``: inputs already resident in HBM, device time from CUDA events on the
decoder's stream, max over ranks.  ``e2e``: the same metric through the public API
(``LayeredDecoder.decode_stream``) from the reference's pageable float64 LLR arrays and
uint8 syndromes to host words, wall-clock per step including every copy.

Multi-GPU (one process per GPU; ``--gpus N`` outside torchrun relaunches itself under
``torch.distributed.run``): every rank decodes its own contiguous frame range
[rank*B, (rank+1)*B) with no collective on the data path; a barrier and a MAX
all-reduce of the timings are the only communication.

``--impl reference`` times the reference's own decoder (the unmodified ``qcldpc``
package installed into baseline/_ref, ThreadPoolExecutor over all host cores; the C
oracle port when it is absent) on a bounded sample of the same workload, on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BATCH = 64
SNR = 0.161
ITERS = 50
SEED = 0
CODE = ROOT / "codes" / "standin_v2_z2500.txt"
# read+write posterior, read+write edge message: FP32 16 B, FP64 32 B, FP16 messages 12 B
BYTES_PER_EDGE_ITER = {"fp32": 16, "fp64": 32, "fp32-msg16": 12}



def single_codeword_l2(latency_ms):
    """L2 traffic of one single-codeword decode from the committed ncu capture
    (tools/single_codeword_profile.py -> profiles/r02_single_codeword_l2.json), over the
    live latency: the decode is bound by its chain of dependent layer steps, not by L2."""
    path = ROOT / "profiles" / "r02_single_codeword_l2.json"
    if not path.exists():
        return {}
    prof = json.loads(path.read_text())
    return {"l2_bytes_per_decode": prof["l2_bytes"], "l2_gbs": prof["l2_bytes"] / latency_ms / 1e6,
            "l2_source": path.name, "launches_profiled": prof["launches"],
            "bound": "dependent layer steps (~3 us each: launch + L2 round trips), L2 throughput "
                     f"{prof['time_weighted_pct_of_peak'].get('lts__t_sectors.avg.pct_of_peak_sustained_elapsed', 0):.1f}% "
                     "of peak under ncu"}

def peaks():
    try:
        p = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in getattr(self, "lines", []):
            f = [x.strip() for x in line.split(",")]
            try:
                sm.append(float(f[1]))
                smax = max(smax, float(f[2]))
            except (ValueError, IndexError):
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def load_code():
    import paper_2004_09084_b200 as q

    base = q.load_base_matrix(CODE)
    sched = q.greedy_schedule(base)
    return base, sched, q.build_compact_index(base, sched)


def cpu_sample(threads, frames, iters, base, sched, index):
    """C oracle (``oracle/layered_ref.c``) decode of `frames` frames x `iters` iterations
    on `threads` threads; returns (Mbit/s at 50 it, seconds)."""
    from oracle import oracle
    import paper_2004_09084_b200 as q

    code = oracle.OracleCode(index, sched)
    n = base.n_cols * base.z
    chan = q.ChannelConfig(snr=SNR, seed=SEED)
    llr = np.stack([q.init_llr(q.transmit(np.zeros(n, np.uint8), chan, q.frame_rng(SEED, 0, i)), chan)
                    for i in range(frames)])
    t0 = time.perf_counter()
    oracle.decode(code, llr, None, iters, False, threads=threads)
    dt = time.perf_counter() - t0
    per_decode = dt * ITERS / iters  # no-ET cost per iteration is constant
    return frames * n / per_decode / 1e6, dt


REF_PKG = ROOT / "baseline" / "_ref"


def reference_package():
    """The unmodified reference package (``qcldpc``) installed into baseline/_ref by
    ``__graft_entry__.build()`` (pip --target from /root/reference), or None."""
    if not (REF_PKG / "qcldpc").is_dir():
        return None
    if str(REF_PKG) not in sys.path:
        sys.path.insert(0, str(REF_PKG))
    try:
        import qcldpc
    except Exception:
        return None
    return qcldpc


class ReferenceSample:
    """The reference's own decode path on host cores: ``qcldpc.LayeredDecoder`` driven
    exactly like ``qcldpc.bench.run_campaign`` (PCG64 frames from ``frame_rng``,
    ``_decode_block`` over a ThreadPoolExecutor of `threads` workers,
    ``/root/reference/pkg/src/qcldpc/bench.py:139-150,216-246``)."""

    def __init__(self, ref, threads, frames):
        from concurrent.futures import ThreadPoolExecutor

        self.ref, self.threads, self.frames = ref, threads, frames
        self.base = ref.load_base_matrix(CODE)
        self.sched = ref.greedy_schedule(self.base)
        self.index = ref.build_compact_index(self.base, self.sched)
        n, m = self.base.n_cols * self.base.z, self.base.n_rows * self.base.z
        self.n = n
        chan = ref.ChannelConfig(snr=SNR, seed=SEED)
        self.llrs = np.empty((frames, n))
        for i in range(frames):
            rng = ref.frame_rng(SEED, 0, i)
            self.llrs[i] = ref.init_llr(ref.transmit(np.zeros(n, np.uint8), chan, rng), chan)
        self.syn = np.zeros((frames, m), np.uint8)
        self.pool = ThreadPoolExecutor(max_workers=threads) if threads > 1 else None

    def run(self, iters):
        """(Mbit/s at 50 iterations, seconds) of one decode of the sample at `iters`."""
        from qcldpc.bench import _decode_block

        dec = self.ref.LayeredDecoder(self.index, self.sched,
                                      self.ref.DecoderConfig(max_iterations=iters, early_termination=False))
        t0 = time.perf_counter()
        _decode_block(dec, self.llrs, self.syn, self.pool, self.threads)
        dt = time.perf_counter() - t0
        return self.frames * self.n / (dt * ITERS / iters) / 1e6, dt


def workload_config(B, frames, world, E, n_layers):
    """The `config` object both arms print (the driver compares them)."""
    return {
        "workload": "configs[2]: 64 codewords/GPU of the rate-0.1 n=1e6 QC-MET-LDPC stand-in, SNR 0.161, "
                    "50 layered iterations, no early termination",
        "code": f"{CODE.name} (360x400 base, z=2500, {E} expanded edges, {n_layers} merged layers)",
        "batch_per_gpu": B, "global_batch": frames, "snr": SNR, "iterations": ITERS,
        "early_termination": False,
        "parallelism": f"dp{world} (independent codeword slices, no collective on the data path)",
        "l2": "per-GPU working set 1.5 GB >> 126 MB L2; no flush between steps",
    }


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle

    base, sched, index = load_code()
    threads = oracle.host_threads()
    frames = threads
    ref = reference_package()
    sample = ReferenceSample(ref, threads, frames) if ref is not None else None
    vals = []
    for step in range(args.warmup + args.steps):
        # one step = a full 50-iteration decode of `frames` frames (no extrapolation)
        v, dt = sample.run(ITERS) if sample else cpu_sample(threads, frames, ITERS, base, sched, index)
        if step >= args.warmup:
            vals.append(v)
    value = float(np.mean(vals))
    port, port_s = cpu_sample(threads, frames, ITERS, base, sched, index)
    kind = "reference" if sample else "port"
    what = ("the unmodified reference package (qcldpc from baseline/_ref: LayeredDecoder via bench._decode_block, "
            f"ThreadPoolExecutor({threads}))" if sample else f"C oracle port on {threads} threads")
    line = {
        "impl": "reference", "metric": "Mbit/s decoded, rate-0.1 n=10^6 QC-MET-LDPC, SNR 0.161, 50 iters",
        "value": value, "unit": "Mbit/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic BIAWGN (reference PCG64 channel), all-zero word, zero syndrome",
        "config": workload_config(BATCH, BATCH * max(args.gpus, 1), max(args.gpus, 1), index.total_edges * base.z,
                                  len(sched.layers)),
        "cpu_baseline": {
            "value": value, "unit": "Mbit/s", "cores": threads, "kind": kind,
            "sample": f"{what}: one full 50-iteration decode of {frames} frames per step",
            "c_port_50it": {"value": port, "seconds": port_s, "frames": frames, "threads": threads},
        },
        "e2e": {"value": value, "unit": "Mbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def read_traffic(kernel, precision="fp32"):
    """Per-launch DRAM bytes of `kernel` (read + write) from the newest committed ncu summary."""
    for p in sorted((ROOT / "profiles").glob("ncu_summary_*.json"), reverse=True):
        try:
            d = json.loads(p.read_text())
            if (d.get("workload") == "configs[2]" and d.get("kernel") == kernel and d.get("dram_bytes_per_launch")
                    and d.get("precision", "fp32") == precision):
                return float(d["dram_bytes_per_launch"]), p.name
        except Exception:
            continue
    return None, None


def run_b200(args):
    world, rank, local = dist_env()
    import torch

    n_dev = torch.cuda.device_count()
    device = local % max(n_dev, 1)  # ranks beyond the visible GPUs share them (plumbing tests only)
    shared = world > n_dev
    torch.cuda.set_device(device)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod

        # NCCL for the barrier and the MAX all-reduce of timings; gloo when ranks share a
        # GPU (NCCL refuses two ranks on one device).  Neither touches the data path.
        if shared:
            dist_mod.init_process_group("gloo")
        else:
            dist_mod.init_process_group("nccl", device_id=torch.device("cuda", device))
        dist = dist_mod
    import paper_2004_09084_b200 as q
    from paper_2004_09084_b200 import _native

    base, sched, index = load_code()
    n, m = base.n_cols * base.z, base.n_rows * base.z
    E = index.total_edges * base.z
    B = args.batch
    cfg = q.DecoderConfig(max_iterations=ITERS, early_termination=False)
    dec = q.LayeredDecoder(index, sched, cfg, device=device, precision=args.precision)
    plan = dec._plan
    st = _native.State(plan, B, args.precision)
    # flow engine with CUDA events around its launch(es), for the roofline; FP64 runs on the
    # per-layer TMA engine (events around every sweep)
    st.set_engine(2 if args.precision == "fp64" else 6)
    st.set_llr_synthetic(seed=SEED, snr_idx=0, first_frame=rank * B, snr=SNR)
    st.set_syndrome(None)
    qcfg = dec._qcfg

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        st.decode(qcfg)
    barrier()
    dev_ms, sweep_ms, launches, layer_launches = [], 0.0, 0, 0
    with Clocks(device) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            dev_ms.append(st.decode(qcfg))
            ll, lms, al = st.kernel_stats()
            sweep_ms += lms
            launches += al
            layer_launches += ll
        barrier()
        wall = time.perf_counter() - t0
    total_ms = float(np.sum(dev_ms))
    _, conv, iters_used = st.results(words=False)
    fer = float((~conv).mean())

    # BASELINE configs[1]: one codeword, the latency of one 50-iteration decode through the
    # default engine choice (one FP32 lane: the per-layer kernels, 1650 dependent launches in
    # one graph with programmatic dependent launch; the 19 MB working set is L2-resident)
    st1 = _native.State(plan, 1, args.precision)
    st1.set_llr_synthetic(seed=SEED, snr_idx=0, first_frame=rank * B, snr=SNR)
    st1.set_syndrome(None)
    b1_ms = [st1.decode(qcfg) for _ in range(3 + max(5, args.steps // 2))][3:]
    b1_launches = st1.kernel_stats()[0]
    del st1

    # e2e through the public API with the reference's own input format: pageable float64
    # (B, n) LLR arrays and uint8 (B, m) syndromes, as run_campaign builds them
    # (/root/reference/pkg/src/qcldpc/bench.py:216-234), words back into host memory.
    # decode_stream overlaps one batch's host conversion + H2D and D2H with the next
    # batch's decode; every step still moves its own inputs and results.
    llr_host = st.get_llr()  # float64 (B, n), the values of the device-resident run
    llr_bufs = [llr_host, llr_host.copy()]
    syn_bufs = [np.zeros((B, m), np.uint8), np.zeros((B, m), np.uint8)]
    del st  # free the device-resident workspace before the streaming slots allocate theirs

    def stream_run(batches, steps):
        for _ in dec.decode_stream([batches(0), batches(1)]):
            pass  # warm the stream workspaces and graphs
        barrier()
        t1 = time.perf_counter()
        for _ in dec.decode_stream((batches(i) for i in range(steps)), depth=2):
            pass
        barrier()
        return (time.perf_counter() - t1) / steps

    e2e_steps = max(3, args.steps)
    e2e_s = stream_run(lambda i: (llr_bufs[i % 2], syn_bufs[i % 2]), e2e_steps)
    # the same stream from pinned float32 buffers (the fastest host format)
    pins = [_native.PinnedArray((B, n), np.float32) for _ in range(2)]
    for p_ in pins:
        p_.array[...] = llr_host
    syn_pin = _native.PinnedArray((B, m), np.uint8)
    syn_pin.array[...] = 0
    pinned_s = stream_run(lambda i: (pins[i % 2].array, syn_pin.array), e2e_steps)
    # the blocking one-call drop-in (decode_batch_arrays) on the reference's pageable
    # float64 arrays (warm: its workspace and graphs are created by the first call)
    dec.decode_batch_arrays(llr_bufs[0], syn_bufs[0])
    t1 = time.perf_counter()
    dec.decode_batch_arrays(llr_bufs[1], syn_bufs[1])
    sync_s = time.perf_counter() - t1

    stats = np.array([total_ms, wall, e2e_s, sweep_ms, pinned_s, sync_s], dtype=np.float64)
    if dist is not None:
        t = torch.tensor(stats, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        stats = t.cpu().numpy()
    total_ms, wall, e2e_s, sweep_ms, pinned_s, sync_s = (float(x) for x in stats)
    if rank != 0:
        return
    frames = world * B
    ms_per_step = total_ms / args.steps
    value = frames * n / (ms_per_step / 1e3) / 1e6
    e2e_value = frames * n / e2e_s / 1e6
    peak, peak_kind = peaks()
    per_launch_ms = sweep_ms / max(layer_launches, 1)
    launches_per_decode = layer_launches / args.steps
    flow = launches_per_decode == 1
    kernel = "flow_kernel" if flow else "layer_tma_kernel"
    # algorithmic bytes of all sweeps of the timed steps, spread over the update-kernel launches
    bpe = BYTES_PER_EDGE_ITER[args.precision]
    alg_bytes_launch = bpe * E * B * ITERS * args.steps / max(layer_launches, 1)
    achieved = alg_bytes_launch / (per_launch_ms / 1e3) / 1e9
    traffic, traffic_src = read_traffic(kernel, args.precision)
    line = {
        "metric": "Mbit/s decoded, rate-0.1 n=10^6 QC-MET-LDPC, SNR 0.161, 50 iters",
        "value": value, "unit": "Mbit/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": {"fp32": "f32", "fp64": "f64", "fp32-msg16": "f32 (f16 edge messages)"}[
            args.precision],
        "data": "synthetic BIAWGN frames generated on device (Philox4x32-10), all-zero word, zero syndrome",
        "config": workload_config(B, frames, world, E, plan.n_layers),
        "fer": fer,
        "precision": args.precision,
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "peak_source": peak_kind, "traffic": traffic, "traffic_source": traffic_src,
            "kernel": ("flow_kernel (one persistent launch per 50-iteration decode, tiles ordered by "
                       "completion flags)") if flow else "layer_tma_kernel (one launch per merged layer unit)",
            "alg_bytes_per_launch": alg_bytes_launch,
            "alg_bytes_note": f"{bpe} B per expanded edge per iteration x {E:,} edges x {B} codewords x 50 "
                              "iterations per decode, divided by the update-kernel launches of a decode",
            "launches_per_decode": launches_per_decode,
            "dram_gbs": (traffic / (per_launch_ms / 1e3) / 1e9) if traffic else None,
            "dram_frac": (traffic / (per_launch_ms / 1e3) / 1e9 / peak) if traffic else None,
            "dram_note": "measured DRAM bytes of one launch (ncu, traffic) / its live duration: the posteriors "
                         "of the 50 high-degree columns stay L2-resident, so DRAM moves ~64% of the algorithmic "
                         "bytes and achieved/peak on algorithmic bytes can exceed 1",
            "avg_launch_ms": per_launch_ms,
            "layer_share_of_step": sweep_ms / max(total_ms, 1e-9),
        },
        "e2e": {
            "value": e2e_value, "unit": "Mbit/s",
            "api": "LayeredDecoder.decode_stream over pageable float64 (B, n) LLR arrays and uint8 (B, m) "
                   "syndromes (the reference's input format), u8 words back to host; the library's host "
                   "threads convert each batch to float32 into pinned chunks while the previous batch decodes",
            "h2d_bytes_per_step": B * n * 4, "d2h_bytes_per_step": B * n + B + 8 * B,
            "bytes_note": "H2D: float32 LLRs after host conversion; the all-zero syndrome is detected on the "
                          "host and not copied",
            "s_per_step": e2e_s, "steps": e2e_steps,
            "pinned_f32_mbit_s": frames * n / pinned_s / 1e6,
            "blocking_call_s": sync_s, "blocking_call_mbit_s": frames * n / sync_s / 1e6,
            "blocking_call_api": "LayeredDecoder.decode_batch_arrays(pageable float64 (64, 10^6), uint8 syndromes)",
        },
        "gpu_launches": int(launches),
        "wall_s_timed": wall,
        "single_codeword": {
            "workload": "configs[1]: one codeword of the same code, SNR 0.161, 50 iterations, no ET",
            "latency_ms": float(np.median(b1_ms)), "latency_ms_min": float(np.min(b1_ms)),
            "mbit_s": n / (float(np.median(b1_ms)) / 1e3) / 1e6, "decodes": len(b1_ms),
            "update_launches_per_decode": int(b1_launches),
            "note": "device time (CUDA events) of qcl_state_decode with the LLRs resident; one-lane layout, "
                    "per-layer kernels in one CUDA graph with programmatic dependent launch (the persistent "
                    "one-launch kernel, QCL_PERSIST=2, measures the same for one FP32 codeword: DESIGN 3.4)",
            **single_codeword_l2(float(np.median(b1_ms))),
        },
    }
    if shared:
        line["ranks_share_gpus"] = f"{world} ranks on {n_dev} visible GPU(s): a plumbing run, not a scaling number"
    line["clocks"] = clk.summary()
    if world == 1:
        from oracle import oracle

        threads = oracle.host_threads()
        ref = reference_package()
        if ref is not None:
            v, dt = ReferenceSample(ref, threads, threads).run(ITERS)
            what, kind = f"the reference package (baseline/_ref qcldpc, ThreadPoolExecutor({threads}))", "reference"
        else:
            v, dt = cpu_sample(threads, threads, ITERS, base, sched, index)
            what, kind = f"C oracle port on {threads} threads", "port"
        line["cpu_baseline"] = {
            "value": v, "unit": "Mbit/s", "cores": threads, "kind": kind,
            "sample": f"{what}: one 50-iteration decode of {threads} frames ({dt:.1f} s)",
        }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def relaunch_cmd(args, port):
    """`python bench.py --gpus N` outside torchrun: one rank per GPU via torch.distributed.run."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()),
            "--gpus", str(args.gpus), "--steps", str(args.steps), "--warmup", str(args.warmup),
            "--batch", str(args.batch), "--impl", args.impl, "--precision", args.precision]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)  # ~0.5 s timed: several clock samples
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--precision", choices=["fp32", "fp64", "fp32-msg16"], default="fp32")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        sys.exit(subprocess.call(relaunch_cmd(args, port)))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()

"""Monte-Carlo decoding campaigns on the device: FER, iterations, latency, throughput.

Mirror of the reference's campaign module (``/root/reference/pkg/src/qcldpc/bench.py``):
the same names (``CampaignConfig``, ``CampaignCell``, ``CampaignReport``,
``ScheduleComparison``, ``run_campaign``, ``compare_schedules``, ``report_to_dict``,
``emit_report``), the same validation messages, the same 8 report columns, CSV/JSON
schema version 1 and metric definitions (``bench.py:51-68,153-185,273-310``), with the
decode running on the B200 path.

Extra ``CampaignConfig`` fields (all optional, reference behaviour by default):

* ``precision`` -- ``"fp32"`` (default, the throughput path), ``"fp64"`` (the parity
  path: the reference's own formula and summation order) or ``"fp32-msg16"`` (opt-in
  FP16 edge messages, flow engine only; FER is compared statistically).
* ``channel`` -- ``"host"`` (default): frames from the reference's PCG64 substreams
  (``frame_rng(seed, snr_idx, frame)``, ``channel.py:36-56``), bit-identical LLRs, so FER
  and iteration counts equal the reference campaign's on the parity path.
  ``"device"``: the same BIAWGN model drawn on the GPU (Philox4x32-10 keyed by
  ``(seed, snr_idx, frame)``, ``csrc/philox.cuh``); no LLR crosses PCIe and frame errors
  are counted on the device (``qcl_state_frame_errors``).  Different noise realisations,
  so FER agrees with the reference's within its confidence interval
  (``tests/test_acceptance.py:194,236`` form), not bit-for-bit.
* ``devices`` -- GPU ordinals; each batch is split into contiguous slices, one per GPU
  and host thread (``np.array_split`` as ``bench.py:143``), no collective.  Default ``(0,)``.
* ``frame_pool`` -- device channel with early termination on the FP32 flow engine: the
  first batch of an SNR point is decoded batched; if its frames stopped on average before
  ~0.85 of the cap, the rest stream through ``batch_size`` lanes per GPU, a lane taking
  the next frame as soon as its frame converges or hits the cap
  (``qcl_state_decode_pool``), so one slow frame no longer holds a batch to the cap;
  otherwise (most frames run to the cap) the rest is decoded batched, where early
  termination runs inside one launch.  Per-frame outcomes, hence FER and average
  iterations, are identical either way; only the timing changes.  Default ``True`` (used
  whenever the flow engine runs; the report's ``roofline`` entries name the path);
  ``"always"`` skips the first-batch probe's choice and streams the rest through the pool.

Timing follows ``bench.py:230-234``: wall-clock around the decode only (LLR generation
and error counting are outside), so ``throughput_mbits_per_s`` is frames * n / decode
seconds / 1e6 at every SNR point.
"""

from __future__ import annotations

import csv
import json
import math
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import asdict, dataclass, field, replace
from pathlib import Path

import numpy as np

from . import _native
from .channel import ChannelConfig, beta, frame_rng, init_llr, transmit
from .decoder import DecoderConfig, LayeredDecoder, syndrome_of
from .layer_schedule import LANE_BUDGET, greedy_schedule, single_row_schedule, utilization
from .qc_code import build_compact_index, descriptor, expand, load_base_matrix

__all__ = [
    "CSV_COLUMNS",
    "METRIC_DEFINITIONS",
    "SCHEMA_VERSION",
    "CampaignCell",
    "CampaignConfig",
    "CampaignReport",
    "ScheduleComparison",
    "compare_schedules",
    "emit_report",
    "report_to_dict",
    "run_campaign",
]

SCHEMA_VERSION = 1

CSV_COLUMNS = (
    "snr",
    "fer",
    "avg_iterations",
    "latency_per_iteration_s",
    "throughput_mbits_per_s",
    "beta",
    "total_expanded_edges",
    "utilization",
)

METRIC_DEFINITIONS = {
    "frame_error": "decoder did not converge, or hard decision differs from the transmitted word",
    "throughput_mbits_per_s": "decoded frames * block_length / decode wall-clock seconds / 1e6",
    "latency_per_iteration_s": "decode wall-clock seconds / total iterations executed",
}

CHANNELS = ("host", "device")


@dataclass(frozen=True)
class CampaignConfig:
    """Everything one campaign needs; validated on construction (``bench.py:71-106``)."""

    matrix_path: str
    snr_list: tuple
    max_iterations: int = 50
    early_termination: bool = False
    batch_size: int = 32
    min_trials: int = 1024
    seed: int = 0
    workers: int = 1
    lane_budget: int = LANE_BUDGET
    encode_mode: bool = False
    merged_schedule: bool = True
    precision: str = "fp32"
    channel: str = "host"
    devices: tuple = (0,)
    frame_pool: bool = True

    def __post_init__(self):
        object.__setattr__(self, "snr_list", tuple(float(s) for s in self.snr_list))
        object.__setattr__(self, "devices", tuple(int(d) for d in self.devices))
        if not self.snr_list:
            raise ValueError("snr_list must not be empty")
        if any(s <= 0 for s in self.snr_list):
            raise ValueError("every snr must be positive")
        if self.batch_size < 1:
            raise ValueError("batch_size must be at least 1")
        if self.min_trials < self.batch_size:
            raise ValueError("min_trials must be at least batch_size")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be at least 1")
        if self.workers < 1:
            raise ValueError("workers must be at least 1")
        if self.lane_budget < 1:
            raise ValueError("lane_budget must be positive")
        if self.precision not in _native.PREC:
            raise ValueError(f"precision must be one of {sorted(_native.PREC)}")
        if self.channel not in CHANNELS:
            raise ValueError(f"channel must be one of {CHANNELS}")
        if not self.devices:
            raise ValueError("devices must not be empty")

    @property
    def frames_per_point(self):
        return math.ceil(self.min_trials / self.batch_size) * self.batch_size


@dataclass(frozen=True)
class CampaignCell:
    """One (snr, configuration) measurement; the 8 report columns."""

    snr: float
    fer: float
    avg_iterations: float
    latency_per_iteration_s: float
    throughput_mbits_per_s: float
    beta: float
    total_expanded_edges: int
    utilization: float


@dataclass(frozen=True)
class CampaignReport:
    cells: tuple
    metadata: dict = field(default_factory=dict)
    # per cell, beside the reference's 8 columns (JSON only): the HBM
    # roofline of the decode at that point (see _roofline)
    roofline: tuple = ()


@dataclass(frozen=True)
class ScheduleComparison:
    """Side-by-side single-row-layer vs merged-layer campaigns."""

    single: CampaignReport
    merged: CampaignReport
    single_layer_count: int
    merged_layer_count: int


def _campaign_metadata(cfg, base, desc, schedule):
    meta = {
        "schema_version": SCHEMA_VERSION,
        "matrix": {
            "path": str(cfg.matrix_path),
            "n_rows": base.n_rows,
            "n_cols": base.n_cols,
            "z": base.z,
            "block_length": desc.block_length,
            "n_checks": desc.n_checks,
            "rate": desc.rate,
        },
        "schedule": {
            "layers": [list(layer) for layer in schedule.layers],
            "layer_count": len(schedule.layers),
            "k1": schedule.k1,
            "merged": cfg.merged_schedule,
        },
        "decoder": {
            "max_iterations": cfg.max_iterations,
            "early_termination": cfg.early_termination,
        },
        "campaign": {
            "batch_size": cfg.batch_size,
            "min_trials": cfg.min_trials,
            "frames_per_point": cfg.frames_per_point,
            "seed": cfg.seed,
            "workers": cfg.workers,
            "lane_budget": cfg.lane_budget,
            "encode_mode": cfg.encode_mode,
        },
        "definitions": dict(METRIC_DEFINITIONS),
    }
    # additive keys only: a reader of schema v1 ignores them
    meta["device"] = {
        "backend": "b200-cuda",
        "precision": cfg.precision,
        "channel": cfg.channel,
        "devices": list(cfg.devices),
        "frame_pool": _uses_pool(cfg),
    }
    return meta


class _HostChannelRunner:
    """Reference frames (bit-identical PCG64 LLRs) through ``decode_batch_arrays``."""

    def __init__(self, cfg, index, schedule, dcfg, n, m, rows):
        self.cfg, self.n, self.m, self.rows = cfg, n, m, rows
        if len(cfg.devices) == 1:
            self.decoders = [LayeredDecoder(index, schedule, dcfg, device=cfg.devices[0], precision=cfg.precision)]
        else:
            self.decoders = [LayeredDecoder(index, schedule, dcfg, device=d, precision=cfg.precision)
                             for d in cfg.devices]
        parts = len(self.decoders) * max(1, cfg.workers)
        self.pool = ThreadPoolExecutor(max_workers=parts) if parts > 1 else None

    def batch(self, snr_idx, chan, start, count):
        cfg, n = self.cfg, self.n
        truths = np.zeros((count, n), dtype=np.uint8)
        llrs = np.empty((count, n))
        for i in range(count):
            rng = frame_rng(cfg.seed, snr_idx, start + i)
            if cfg.encode_mode:
                truths[i] = rng.integers(0, 2, size=n, dtype=np.uint8)
            llrs[i] = init_llr(transmit(truths[i], chan, rng), chan)
        if cfg.encode_mode:
            syndromes = syndrome_of(truths, self.rows)
        else:
            syndromes = np.zeros((count, self.m), dtype=np.uint8)

        t0 = time.perf_counter()
        words, converged, iterations = self._decode(llrs, syndromes)
        wall = time.perf_counter() - t0
        mismatch = (words != truths).any(axis=1)
        return converged, mismatch, iterations, wall

    def _decode(self, llrs, syndromes):
        if self.pool is None:
            return self.decoders[0].decode_batch_arrays(llrs, syndromes)
        # contiguous slices: devices first, then the reference's worker split per device
        jobs = []
        for d, dev_rows in zip(self.decoders, np.array_split(np.arange(llrs.shape[0]), len(self.decoders))):
            for c in np.array_split(dev_rows, max(1, self.cfg.workers)):
                if c.size:
                    jobs.append((d, c))
        parts = list(self.pool.map(lambda j: j[0].decode_batch_arrays(llrs[j[1]], syndromes[j[1]]), jobs))
        return tuple(np.concatenate([p[k] for p in parts]) for k in range(3))

    def close(self):
        if self.pool is not None:
            self.pool.shutdown()


class _DeviceChannelRunner:
    """Frames drawn on each GPU (Philox), decoded in place; only flags come back."""

    def __init__(self, cfg, index, schedule, dcfg, n, m, rows):
        self.cfg = cfg
        self.qcfg = _native.make_config(dcfg, cfg.precision)
        self.plans = [_native.Plan(index, schedule, d) for d in cfg.devices]
        self.states = {}
        self.pool = ThreadPoolExecutor(max_workers=len(self.plans)) if len(self.plans) > 1 else None

    def _state(self, dev, count):
        key = (dev, count)
        if key not in self.states:
            st = _native.State(self.plans[dev], count, self.cfg.precision)
            # one untimed decode: the engine's one-time set-up (tile tables, flags, the decode
            # graph) stays out of the first SNR point's timing
            st.set_llr_synthetic(self.cfg.seed, 0, 0, 1.0)
            st.set_syndrome(None)
            st.decode(self.qcfg)
            self.states[key] = st
        return self.states[key]

    def _slice(self, job):
        dev, snr_idx, snr, first, count = job
        st = self._state(dev, count)
        st.set_llr_synthetic(self.cfg.seed, snr_idx, first, snr, encode_mode=self.cfg.encode_mode)
        t0 = time.perf_counter()
        st.decode(self.qcfg)
        _, converged, iterations = st.results(words=False)
        wall = time.perf_counter() - t0
        return converged, st.frame_errors(), iterations, wall

    def batch(self, snr_idx, chan, start, count):
        sizes = [len(c) for c in np.array_split(np.arange(count), len(self.plans))]
        jobs, first = [], start
        for dev, size in enumerate(sizes):
            if size:
                jobs.append((dev, snr_idx, chan.snr, first, size))
            first += size
        parts = list(self.pool.map(self._slice, jobs)) if self.pool else [self._slice(j) for j in jobs]
        converged = np.concatenate([p[0] for p in parts])
        mismatch = np.concatenate([p[1] for p in parts])
        iterations = np.concatenate([p[2] for p in parts])
        return converged, mismatch, iterations, max(p[3] for p in parts)

    def close(self):
        if self.pool is not None:
            self.pool.shutdown()


def _uses_pool(cfg):
    return (cfg.frame_pool and cfg.channel == "device" and cfg.early_termination and not cfg.encode_mode
            and cfg.precision in ("fp32", "fp32-msg16"))


class _PoolRunner(_DeviceChannelRunner):
    """All frames of an SNR point through ``batch_size`` lanes per GPU (frame pool)."""

    def _jobs(self, snr_idx, snr, frames):
        sizes = [len(c) for c in np.array_split(np.arange(frames), len(self.plans))]
        jobs, first = [], 0
        for dev, size in enumerate(sizes):
            if size:
                jobs.append((dev, snr_idx, snr, first, size))
            first += size
        return jobs

    def supported(self, frames):
        """The pool needs the flow engine for every per-GPU lane set (>= 4 lanes, row
        degree <= 12, tables in shared memory): asked of the engine itself."""
        return all(self._state(dev, min(self.cfg.batch_size, count)).info()[1]
                   for dev, _, _, _, count in self._jobs(0, 1.0, frames))

    # The pool pays ~0.71 ms per 64-lane sweep (a launch per sweep plus refills), a batched
    # decode ~0.52 ms (early termination fused into one launch, DESIGN 3.3) but every sweep
    # until the batch's slowest frame is done -- the cap as soon as one frame fails.  Measured
    # on the n = 1e6 stand-in (profiles/r02_campaign_sweep_*.json, caps 20/50/100, SNR
    # 0.14-0.20) the pool wins when frames stop on average before ~0.85 of the cap.
    POOL_WHEN_MEAN_BELOW = 0.85

    def point(self, snr_idx, chan, frames):
        """All frames of one SNR point: the first batch as a batched decode, the rest in the
        frame pool when that batch's mean iteration count says the pool pays, else as
        further batches.  Frames are independent, so every frame's outcome is the same
        whichever path decodes it; only the timing differs.  Returns (converged, frame
        error, iterations, wall seconds, path)."""
        first = min(self.cfg.batch_size * len(self.plans), frames)
        parts = [self.batch(snr_idx, chan, 0, first)]
        use_pool = (self.cfg.frame_pool == "always"
                    or float(parts[0][2].mean()) < self.POOL_WHEN_MEAN_BELOW * self.cfg.max_iterations)
        if frames > first and use_pool:
            jobs = [(dev, si, snr, f0 + first, count) for dev, si, snr, f0, count
                    in self._jobs(snr_idx, chan.snr, frames - first)]

            def run(job):
                dev, si, snr, f0, count = job
                st = self._state(dev, min(self.cfg.batch_size, count))
                t0 = time.perf_counter()
                conv, iters, err, _ = st.decode_pool(self.qcfg, self.cfg.seed, si, f0, count, snr)
                return conv, err, iters, time.perf_counter() - t0

            rest = list(self.pool.map(run, jobs)) if self.pool else [run(j) for j in jobs]
            parts.append((np.concatenate([r[0] for r in rest]), np.concatenate([r[1] for r in rest]),
                          np.concatenate([r[2] for r in rest]), max(r[3] for r in rest)))
        else:
            for start in range(first, frames, self.cfg.batch_size):
                parts.append(self.batch(snr_idx, chan, start, min(self.cfg.batch_size, frames - start)))
        return (np.concatenate([x[0] for x in parts]), np.concatenate([x[1] for x in parts]),
                np.concatenate([x[2] for x in parts]), sum(x[3] for x in parts),
                "pool" if (frames > first and use_pool) else "batched")


BYTES_PER_EDGE_ITERATION = {"fp32": 16, "fp64": 32, "fp32-msg16": 12}


def _hbm_peak():
    """Per-GPU HBM bandwidth the fractions refer to: MEASURED_PEAKS.json (driver-written,
    next to the package) when present, else the B200 profiling recipe's fallback."""
    try:
        peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
        return float(peaks["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _device_metadata(cfg, pool):
    import os

    peak, source = _hbm_peak()
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        cores = os.cpu_count()
    return {
        "precision": cfg.precision,
        "channel": cfg.channel,
        "devices": list(cfg.devices),
        "gpu_count": len(set(cfg.devices)),
        "host_cores": cores,
        "frame_pool": bool(pool),
        "bytes_per_edge_iteration": BYTES_PER_EDGE_ITERATION[cfg.precision],
        "hbm_peak_gbs_per_gpu": peak,
        "hbm_peak_source": source,
    }


def _roofline(cell, iterations_total, wall, device_meta):
    """Algorithmic HBM bytes of the decode at one SNR point (bytes per edge-iteration x
    expanded edges x iterations executed, summed over frames) over its decode wall time,
    per GPU and as a fraction of the per-GPU peak."""
    bpe = device_meta["bytes_per_edge_iteration"]
    edge_iterations = int(iterations_total) * int(cell.total_expanded_edges)
    achieved = bpe * edge_iterations / wall / 1e9 if wall > 0 else 0.0
    per_gpu = achieved / max(1, device_meta["gpu_count"])
    return {
        "snr": cell.snr,
        "edge_iterations": edge_iterations,
        "achieved_gbs": achieved,
        "achieved_gbs_per_gpu": per_gpu,
        "roofline_fraction": per_gpu / device_meta["hbm_peak_gbs_per_gpu"],
        "bytes_per_edge_iteration": bpe,
    }


def run_campaign(cfg):
    """Measure FER/iterations/latency/throughput at every SNR point (``bench.py:188-258``)."""
    base = load_base_matrix(cfg.matrix_path)
    desc = descriptor(base)
    schedule = greedy_schedule(base) if cfg.merged_schedule else single_row_schedule(base)
    index = build_compact_index(base, schedule)
    dcfg = DecoderConfig(max_iterations=cfg.max_iterations, early_termination=cfg.early_termination)
    rows = expand(base) if (cfg.encode_mode and cfg.channel == "host") else None
    util = utilization(schedule, k2=cfg.batch_size, z=base.z, lane_budget=cfg.lane_budget)

    n = desc.block_length
    m = desc.n_checks
    frames = cfg.frames_per_point
    pool = _uses_pool(cfg)
    runner_cls = _PoolRunner if pool else (_HostChannelRunner if cfg.channel == "host" else _DeviceChannelRunner)
    runner = runner_cls(cfg, index, schedule, dcfg, n, m, rows)
    if pool and not runner.supported(frames):
        pool = False  # the batched device-channel decode (a _PoolRunner is one) runs instead

    cells, roofline = [], []
    try:
        for snr_idx, snr in enumerate(cfg.snr_list):
            chan = ChannelConfig(snr=snr, seed=cfg.seed)
            errors = 0
            iterations_total = 0
            wall = 0.0
            path = "batched"
            if pool:
                converged, mismatch, iterations, wall, path = runner.point(snr_idx, chan, frames)
                errors += int((~converged).sum()) + int((converged & mismatch).sum())
                iterations_total += int(iterations.sum())
            for start in range(0, 0 if pool else frames, cfg.batch_size):
                batch = min(cfg.batch_size, frames - start)
                converged, mismatch, iterations, dt = runner.batch(snr_idx, chan, start, batch)
                wall += dt
                errors += int((~converged).sum())
                errors += int((converged & mismatch).sum())
                iterations_total += int(iterations.sum())
            cells.append(
                CampaignCell(
                    snr=snr,
                    fer=errors / frames,
                    avg_iterations=iterations_total / frames,
                    latency_per_iteration_s=wall / iterations_total,
                    throughput_mbits_per_s=frames * n / wall / 1e6,
                    beta=beta(desc.rate, snr),
                    total_expanded_edges=desc.total_expanded_edges,
                    utilization=util.utilization,
                )
            )
            roofline.append((iterations_total, wall, path))
    finally:
        runner.close()

    metadata = _campaign_metadata(cfg, base, desc, schedule)
    metadata["device"] = _device_metadata(cfg, pool)
    return CampaignReport(cells=tuple(cells), metadata=metadata,
                          roofline=tuple(dict(_roofline(c, it, w, metadata["device"]), path=path)
                                         for c, (it, w, path) in zip(cells, roofline)))


def compare_schedules(cfg):
    """Run the same campaign with single-row layers and with merged layers (``bench.py:261-270``)."""
    single = run_campaign(replace(cfg, merged_schedule=False))
    merged = run_campaign(replace(cfg, merged_schedule=True))
    return ScheduleComparison(
        single=single,
        merged=merged,
        single_layer_count=single.metadata["schedule"]["layer_count"],
        merged_layer_count=merged.metadata["schedule"]["layer_count"],
    )


def report_to_dict(report):
    if isinstance(report, ScheduleComparison):
        return {
            "schema_version": SCHEMA_VERSION,
            "single": report_to_dict(report.single),
            "merged": report_to_dict(report.merged),
            "single_layer_count": report.single_layer_count,
            "merged_layer_count": report.merged_layer_count,
        }
    out = {
        "schema_version": SCHEMA_VERSION,
        "metadata": report.metadata,
        "cells": [asdict(cell) for cell in report.cells],
    }
    if report.roofline:
        out["roofline"] = list(report.roofline)
    return out


def emit_report(report, fmt, path):
    """Write a campaign report (or comparison) as csv or json (``bench.py:289-310``)."""
    path = Path(path)
    if fmt == "json":
        path.write_text(json.dumps(report_to_dict(report), indent=2) + "\n")
        return path
    if fmt != "csv":
        raise ValueError(f"unknown report format {fmt!r}")

    comparison = isinstance(report, ScheduleComparison)
    header = (("schedule",) + CSV_COLUMNS) if comparison else CSV_COLUMNS
    with path.open("w", newline="") as fh:
        writer = csv.writer(fh, lineterminator="\n")
        writer.writerow(header)
        reports = (("single", report.single), ("merged", report.merged)) if comparison else ((None, report),)
        for label, rep in reports:
            for cell in rep.cells:
                row = tuple(asdict(cell)[c] for c in CSV_COLUMNS)
                writer.writerow(((label,) + row) if comparison else row)
    return path


def main(argv=None):
    """``python -m paper_2004_09084_b200.campaign``: the ``decode-bench run`` /
    ``compare-schedules`` campaign (reference ``cli.py:94-139``) on the device."""
    import argparse

    ap = argparse.ArgumentParser(prog="python -m paper_2004_09084_b200.campaign")
    ap.add_argument("--matrix", required=True)
    ap.add_argument("--snr", type=float, nargs="+", required=True)
    ap.add_argument("--iterations", type=int, default=50)
    ap.add_argument("--early-termination", action="store_true")
    ap.add_argument("--batch-size", type=int, default=32)
    ap.add_argument("--min-trials", type=int, default=1024)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--encode-mode", action="store_true")
    ap.add_argument("--single-row", action="store_true", help="one base row per layer")
    ap.add_argument("--precision", choices=sorted(_native.PREC), default="fp32")
    ap.add_argument("--channel", choices=CHANNELS, default="host")
    ap.add_argument("--devices", type=int, nargs="+", default=[0])
    ap.add_argument("--compare-schedules", action="store_true")
    ap.add_argument("--format", choices=("csv", "json"), default="json")
    ap.add_argument("--out", required=True)
    a = ap.parse_args(argv)
    cfg = CampaignConfig(
        matrix_path=a.matrix, snr_list=a.snr, max_iterations=a.iterations, early_termination=a.early_termination,
        batch_size=a.batch_size, min_trials=a.min_trials, seed=a.seed, workers=a.workers,
        encode_mode=a.encode_mode, merged_schedule=not a.single_row, precision=a.precision, channel=a.channel,
        devices=a.devices,
    )
    report = compare_schedules(cfg) if a.compare_schedules else run_campaign(cfg)
    emit_report(report, a.format, a.out)
    cells = report.merged.cells if a.compare_schedules else report.cells
    for c in cells:
        print(f"snr {c.snr:g}: fer {c.fer:.6g}, avg iterations {c.avg_iterations:.3f}, "
              f"{c.throughput_mbits_per_s:.1f} Mbit/s")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())

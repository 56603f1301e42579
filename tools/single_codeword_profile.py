"""configs[1] (one codeword, n = 10^6, 50 iterations): which resource bounds the latency.

    ncu --profile-from-start off --clock-control none --csv --log-file gpurun_out/sc.csv \
        --metrics gpu__time_duration.sum,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
        lts__t_sectors.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed \
        python tools/single_codeword_profile.py
    python tools/single_codeword_profile.py --summarize gpurun_out/sc.csv > profiles/r02_single_codeword_l2.json
    (QCL_PERSIST=0: the per-layer graph, r02_single_codeword_l2.json; default: the persistent
    kernel, r02_single_codeword_persist_l2.json, read by bench.py)

The first mode decodes one codeword twice and opens the profiler range around the second
decode only (every launch of one decode).  The second mode sums the per-launch metrics.
"""
import csv
import json
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

if len(sys.argv) > 2 and sys.argv[1] == "--summarize":
    rows = []
    with open(sys.argv[2]) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    per = defaultdict(lambda: defaultdict(float))
    launches = defaultdict(set)
    units = {}
    dur = {r["ID"]: float(r["Metric Value"].replace(",", "")) * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(
        r["Metric Unit"], 1) for r in rows if r["Metric Name"] == "gpu__time_duration.sum"}
    pct = defaultdict(float)  # time-weighted mean of the percent-of-peak metrics
    for r in rows:
        if "pct" in r["Metric Name"]:
            pct[r["Metric Name"]] += float(r["Metric Value"].replace(",", "")) * dur.get(r["ID"], 0.0)
            continue
        k = r["Kernel Name"].split("(")[0].split("<")[0]
        launches[k].add(r["ID"])
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(unit, 1)
        per[k][r["Metric Name"]] += v * scale
        units[r["Metric Name"]] = "ns" if "time" in r["Metric Name"] else "bytes"
    tot = defaultdict(float)
    for k in per:
        for mname, v in per[k].items():
            tot[mname] += v
    n_launch = sum(len(v) for v in launches.values())
    t_ns = tot["gpu__time_duration.sum"]
    out = {
        "workload": "configs[1]: one codeword, standin_v2_z2500, SNR 0.161, 50 iterations, no ET, FP32, "
                    + ("persistent per-layer kernel (one cooperative launch)" if any("layer_persist_kernel" in k for k in per)
                       else "per-layer graph"),
        "launches": n_launch,
        "serialized_kernel_ms": t_ns / 1e6,
        "l2_bytes": tot["lts__t_bytes.sum"],
        "dram_bytes": tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"],
        "l2_gbs_over_kernel_time": tot["lts__t_bytes.sum"] / t_ns,
        "mean_launch_us": t_ns / 1e3 / max(n_launch, 1),
        "time_weighted_pct_of_peak": {m: v / t_ns for m, v in pct.items()},
        "per_kernel": {k: {"launches": len(launches[k]), **{m: v for m, v in per[k].items()}} for k in per},
        "note": "ncu serialises launches (and drops the programmatic-dependent-launch overlap of the "
                "per-layer graph); durations are cold per launch. L2 bytes and DRAM bytes are per decode.",
    }
    print(json.dumps(out, indent=1))
    sys.exit(0)

import torch  # noqa: E402

import paper_2004_09084_b200 as q  # noqa: E402
from paper_2004_09084_b200 import _native  # noqa: E402

base = q.load_base_matrix(ROOT / "codes" / "standin_v2_z2500.txt")
sched = q.greedy_schedule(base)
plan = _native.Plan(q.build_compact_index(base, sched), sched, 0)
cfg = _native.make_config(q.DecoderConfig(max_iterations=50, early_termination=False), "fp32")
st = _native.State(plan, 1, "fp32")
st.set_llr_synthetic(seed=0, snr_idx=0, first_frame=0, snr=0.161)
st.set_syndrome(None)
print(f"warm decode: {st.decode(cfg):.2f} ms", flush=True)
torch.cuda.profiler.start()
ms = st.decode(cfg)
torch.cuda.profiler.stop()
print(f"profiled decode: {ms:.2f} ms (under the profiler)", flush=True)

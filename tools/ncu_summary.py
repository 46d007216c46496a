"""Extract the roofline-relevant counters from `ncu --set full` reports into
profiles/ncu_summary.json (+ a readable .md). Usage:
    python tools/ncu_summary.py OUT_PREFIX name=report.ncu-rep:m,n,k[:op] ...
(shape prefixes: s = operand split rows,cols pairs; g = GEMV-class m,n,k in GB/s)
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_tc_pipe_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "registers",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_scoreboard",
}
UNIT = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
        "s": 1.0, "second": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "Hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}


def read(rep, pattern=None):
    import re

    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    vals = next(r for r in rows[2:] if pattern is None or re.search(pattern, r[ki]))
    res = {"kernel": vals[hdr.index("Kernel Name")]}
    for k, name in KEYS.items():
        if k in hdr:
            i = hdr.index(k)
            v = float(vals[i].replace(",", ""))
            res[name] = v * UNIT.get(units[i], 1.0) if units[i] in UNIT else v
    return res


def main(prefix, specs):
    summary = {}
    md = ["| capture | kernel | time | DRAM read+write | algorithmic | tensor pipe | DRAM % | L2 hit | achieved |",
          "|---|---|---|---|---|---|---|---|---|"]
    for spec in specs:
        name, rest = spec.split("=", 1)
        rep, shape = rest.split(":", 1)
        parts = shape.split(":")
        r = read(rep, parts[1] if len(parts) > 1 else None)
        r["traffic_bytes"] = r.get("dram_read", 0) + r.get("dram_write", 0)
        split = parts[0].startswith("s")
        gemv = parts[0].startswith("g")  # GEMV-class product: HBM-bound, report GB/s
        dims = [int(x) for x in parts[0].lstrip("sg").split(",")]
        if gemv:
            m, n, k = dims
            r["algorithmic_bytes"] = 4 * (m * k + n * k + m * n)
            r["achieved"] = f"{r['algorithmic_bytes'] / r['duration'] / 1e9:.0f} GB/s"
        elif split:
            # operand split: read x (4 B), write h + l (2 B + 2 B) per element
            r["algorithmic_bytes"] = 8 * sum(dims[i] * dims[i + 1] for i in range(0, len(dims), 2))
            r["achieved"] = f"{r['algorithmic_bytes'] / r['duration'] / 1e9:.0f} GB/s"
        elif len(dims) == 3:
            m, n, k = dims
            # hi/lo halves of A and B (4 bytes per element in total for both the
            # TF32 lo-only and the FP16 h+l splits, plus the raw fp32 operand read as
            # hi by the TF32 kind) and C; report the FP16 kind's: 4(mk + nk) + 4mn
            r["algorithmic_bytes"] = 4 * (m * k + n * k + m * n)
            r["achieved"] = f"{2 * m * n * k / r['duration'] / 1e12:.1f} TFLOP/s"
        elif len(dims) == 2:
            rr, cc = dims
            r["algorithmic_bytes"] = 8 * rr * cc
            r["achieved"] = f"{8 * rr * cc / r['duration'] / 1e9:.0f} GB/s"
        summary[name] = r
        md.append(f"| {name} | {r['kernel'][:40]} | {r['duration']*1e3:.3f} ms | "
                  f"{r['traffic_bytes']/1e9:.2f} GB | {r['algorithmic_bytes']/1e9:.2f} GB | "
                  f"{r.get('tensor_pipe_pct', 0):.1f}% | {r.get('dram_pct', 0):.1f}% | "
                  f"{r.get('l2_hit_pct', 0):.1f}% | {r['achieved']} |")
    json.dump(summary, open(prefix + ".json", "w"), indent=1)
    open(prefix + ".md", "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])

"""Summarise an ncu report (--set full) and a launch list into profiles/.

    python tools/ncu_summary.py gpurun_out/prof_r1.ncu-rep gpurun_out/launches.csv r01

writes profiles/r01_ncu_summary.json / .md and profiles/traffic.json (DRAM
bytes per launch of each kernel, read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "lts__t_bytes.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return v * scale


def main():
    reps, launches, tag = sys.argv[1].split(","), sys.argv[2], sys.argv[3]
    per = defaultdict(list)
    for rep in reps:
        hdr, units, data = raw(rep)
        collect(hdr, units, data, per)
    finish(",".join(reps), per, launches, tag)


def collect(hdr, units, data, per):
    ik = hdr.index("Kernel Name")
    for r in data:
        name = r[ik].split("(")[0].replace("void ", "").strip()
        d = {}
        for m in METRICS:
            if m in hdr:
                j = hdr.index(m)
                val = r[j]
                if m.startswith("dram__bytes") or m == "lts__t_bytes.sum":
                    d[m] = to_bytes(val, units[j])
                elif m == "gpu__time_duration.sum":
                    t = float(val.replace(",", ""))
                    d["duration_us"] = t / 1e3 if units[j].startswith("n") else (t if units[j].startswith("u") else t * 1e3)
                else:
                    try:
                        d[m] = float(val.replace(",", ""))
                    except ValueError:
                        d[m] = val
        per[name].append(d)


def finish(rep, per, launches, tag):
    summary = {}
    for name, lst in per.items():
        avg = {k: sum(x[k] for x in lst if isinstance(x.get(k), float)) / len(lst) for k in lst[0]}
        avg["dram_bytes_per_launch"] = avg.get("dram__bytes_read.sum", 0) + avg.get("dram__bytes_write.sum", 0)
        avg["captured_launches"] = len(lst)
        summary[name] = avg
    # launch list shares
    shares = defaultdict(float)
    total = 0.0
    with open(launches) as fh:
        lines = [ln for ln in fh if not ln.startswith("==")]
    rd = csv.reader(lines)
    hdr2 = next(rd)
    kn, mv, mn = hdr2.index("Kernel Name"), hdr2.index("Metric Value"), hdr2.index("Metric Name")
    counts = defaultdict(int)
    for r in rd:
        if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
            continue
        name = r[kn].split("(")[0].replace("void ", "").strip()
        t = float(r[mv].replace(",", ""))
        shares[name] += t
        counts[name] += 1
        total += t
    launch_share = {k: {"launches": counts[k], "total_ms": v / 1e6, "share": v / total}
                    for k, v in sorted(shares.items(), key=lambda kv: -kv[1])}
    out = {"report": rep, "kernels": summary, "launch_list": launch_share,
           "note": "ncu --set full --clock-control none (per-launch replays: cold-cache, serialised); "
                   "compare shares, not absolutes"}
    prof = Path(__file__).resolve().parents[1] / "profiles"
    prof.mkdir(exist_ok=True)
    (prof / f"{tag}_ncu_summary.json").write_text(json.dumps(out, indent=1))
    traffic = {}
    for name, avg in summary.items():
        base = name.split("<")[0].split("::")[-1]
        traffic[base] = avg["dram_bytes_per_launch"]
    (prof / "traffic.json").write_text(json.dumps(traffic, indent=1))
    md = [f"# ncu summary {tag}", "", f"report: `{rep}` (ncu --set full, --clock-control none)", "",
          "| kernel | launches captured | duration us | DRAM bytes/launch | DRAM GB/s | DRAM % peak | SM % | "
          "issue active % | regs |",
          "|---|---|---|---|---|---|---|---|---|"]
    for name, a in sorted(summary.items(), key=lambda kv: -kv[1].get("duration_us", 0)):
        dur = a.get("duration_us", 0) or 1e-9
        md.append(f"| {name} | {a['captured_launches']} | {a.get('duration_us', 0):.1f} | "
                  f"{a['dram_bytes_per_launch'] / 1e6:.1f} MB | {a['dram_bytes_per_launch'] / dur / 1e3:.0f} | "
                  f"{a.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                  f"{a.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                  f"{a.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                  f"{a.get('launch__registers_per_thread', 0):.0f} |")
    md += ["", "## launch list (`ncu --metrics gpu__time_duration.sum --clock-control none` over `python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline`, every launch incl. frame 1 and clip synthesis)", "",
           "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in launch_share.items():
        md.append(f"| {k} | {v['launches']} | {v['total_ms']:.2f} | {100 * v['share']:.1f}% |")
    (prof / f"{tag}_ncu_summary.md").write_text("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()

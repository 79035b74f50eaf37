"""Summarise an ncu launch list + full capture into profiles/ (markdown + json).

python tools/summarize_ncu.py r1   (reads gpurun_out/launches_r1.csv, full_raw_r1.csv, full_src_r1.csv)
"""
import csv
import io
import json
import os
import sys
from collections import defaultdict

R = sys.argv[1] if len(sys.argv) > 1 else "r1"
OUT = "profiles"
os.makedirs(OUT, exist_ok=True)


def short(name):
    name = name.replace("rtpb::", "").replace("(rtpb::GemmMaps, rtpb::GemmArgs)", "")
    return name[:110]


lines = []
# ---- launch list: share of device time per kernel over the captured bench command
agg = defaultdict(lambda: [0, 0.0])
try:
    rows = list(csv.reader(open(f"gpurun_out/launches_{R}.csv")))
    hdr = None
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(
                    d.get("Metric Unit", "nsecond"), 1e-3)
                agg[short(d["Kernel Name"])][0] += 1
                agg[short(d["Kernel Name"])][1] += float(d["Metric Value"].replace(",", "")) * scale  # us
except FileNotFoundError:
    pass
tot = sum(v[1] for v in agg.values()) or 1.0
lines.append(f"# ncu summary {R}\n")
lines.append("## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, bench.py --steps 3)\n")
lines.append("Cold-cache, serialised per-launch times: compare shares, not absolutes.\n")
lines.append("| share | launches | avg us | kernel |\n|---:|---:|---:|---|")
ours = 0.0
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"| {100 * v[1] / tot:.1f}% | {v[0]} | {v[1] / v[0]:.1f} | `{k}` |")
    if "rtp_gemm" in k or "colsum" in k or "flyweight" in k:
        ours += v[1]
lines.append(f"\nLibrary kernels: {100 * ours / tot:.1f}% of device time in the captured command "
             "(the rest is the bench harness: L2 flush, input generation).\n")

# ---- full capture: per-kernel metrics
summary = {"round": R, "kernels": []}
try:
    rows = list(csv.reader(open(f"gpurun_out/full_raw_{R}.csv")))
    hdr = rows[0]
    units = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}

    def g(r, key):
        for h in hdr:
            if h == key or h.endswith("." + key) or h.endswith(key):
                return r[idx[h]], units[idx[h]]
        return None, None

    lines.append("## Full capture (`ncu --set full`, step GEMMs)\n")
    lines.append("| kernel | grid | time us | tensor pipe % | L2 % | SM MHz | DRAM read MB | DRAM write MB | issue % | regs |")
    lines.append("|---|---|---:|---:|---:|---:|---:|---:|---:|---:|")
    for r in rows[2:]:
        name = short(r[idx["Kernel Name"]])
        t, tu = g(r, "gpu__time_duration.sum")
        if t:  # normalise to microseconds whatever unit ncu chose
            t = str(float(t) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
                                "ms": 1e3, "second": 1e6, "s": 1e6}.get(tu, 1.0))
        tp, _ = g(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
        dr, dru = g(r, "dram__bytes_read.sum")
        dw, dwu = g(r, "dram__bytes_write.sum")
        iss, _ = g(r, "sm__inst_issued.avg.pct_of_peak_sustained_active")
        regs, _ = g(r, "launch__registers_per_thread")
        l2, _ = g(r, "lts__throughput.avg.pct_of_peak_sustained_elapsed")
        clk, clku = g(r, "sm__cycles_elapsed.avg.per_second")
        grid, _ = g(r, "Grid Size")

        def mb(v, u):
            try:
                v = float(v)
            except (TypeError, ValueError):
                return None
            return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
        rec = {"kernel": name, "grid": grid, "time_us": float(t) if t else None,
               "tensor_pipe_pct": float(tp) if tp else None, "dram_read_MB": mb(dr, dru),
               "dram_write_MB": mb(dw, dwu), "issue_pct": float(iss) if iss else None, "regs": regs,
               "l2_pct": float(l2) if l2 else None,
               "sm_mhz": (float(clk) * {"Ghz": 1e3, "hz": 1e-6, "Khz": 1e-3, "Mhz": 1.0}.get(clku, 1.0)) if clk else None}
        summary["kernels"].append(rec)
        lines.append(f"| `{name[:70]}` | {grid} | {rec['time_us']:.1f} | {rec['tensor_pipe_pct'] or 0:.1f} | {rec['l2_pct'] or 0:.1f} | {rec['sm_mhz'] or 0:.0f} | "
                     f"{rec['dram_read_MB'] or 0:.1f} | {rec['dram_write_MB'] or 0:.1f} | {rec['issue_pct'] or 0:.1f} "
                     f"| {regs} |")
except (FileNotFoundError, IndexError):
    pass

# ---- source page: top stall reasons per kernel
try:
    text = open(f"gpurun_out/full_src_{R}.csv").read().split("\n")
    secs, cur = [], None
    for ln in text:
        if ln.startswith('"Kernel Name"'):
            cur = [ln]
            secs.append(cur)
        elif cur is not None:
            cur.append(ln)
    lines.append("\n## Warp-stall samples (source page, top reasons per kernel)\n")
    seen = set()
    for sec in secs:
        name = short(sec[0].split(",", 1)[1].strip('",'))
        if name in seen:
            continue
        seen.add(name)
        rdr = list(csv.reader(io.StringIO("\n".join(sec[1:]))))
        h = rdr[0]
        ix = {k: i for i, k in enumerate(h)}
        data = [r for r in rdr[1:] if len(r) == len(h)]
        cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
        aggs = {c: sum(int(r[ix[c]] or 0) for r in data) for c in cols}
        top = sorted(((v, c) for c, v in aggs.items()), reverse=True)[:5]
        lines.append(f"* `{name[:80]}`: " + ", ".join(f"{c[6:]} {v}" for v, c in top))
except FileNotFoundError:
    pass

open(f"{OUT}/ncu_{R}.md", "w").write("\n".join(lines) + "\n")
json.dump(summary, open(f"{OUT}/ncu_{R}.json", "w"), indent=1)
# dominant-kernel DRAM traffic per launch, for bench.py's roofline.traffic
# (keyed by bench config: CONFIG env, default d)
ks = [k for k in summary["kernels"] if k["time_us"]]
if ks:
    avg = sum((k["dram_read_MB"] or 0) + (k["dram_write_MB"] or 0) for k in ks) / len(ks)
    cfg = os.environ.get("CONFIG", "d")
    path = f"{OUT}/ncu_traffic.json"
    try:
        tj = json.load(open(path))
    except (FileNotFoundError, ValueError):
        tj = {}
    tj.setdefault("configs", {})[cfg] = {
        "source": f"profiles/ncu_{R}.md", "kernel": "rtp_gemm_kernel (step GEMMs, average over captured launches)",
        "dram_bytes_per_launch": avg * 1e6, "launches": len(ks),
        "per_launch_MB": [round((k["dram_read_MB"] or 0) + (k["dram_write_MB"] or 0), 1) for k in ks]}
    json.dump(tj, open(path, "w"), indent=1)
print("\n".join(lines))

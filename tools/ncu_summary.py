"""Markdown summary of ncu --set full reports: per kernel launch duration, DRAM traffic,
throughputs, occupancy, tensor pipe, top stall reasons.
usage: python tools/ncu_summary.py rep1.ncu-rep [rep2 ...] > summary.md"""
import csv, io, subprocess, sys, json

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read_B",
    "dram__bytes_write.sum": "dram_write_B",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "regs",
    "smsp__inst_executed.sum": "warp_insts",
    "lts__t_bytes.sum": "l2_bytes",
}
UNIT = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for line in r[2:]:
        d = dict(zip(hdr, line))
        u = dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name", "")[:60]}
        for k, name in KEYS.items():
            if k in d:
                try:
                    v = float(d[k].replace(",", ""))
                    if name == "duration_us":
                        v *= UNIT.get(u.get(k, "usecond"), 1.0)
                    elif name.endswith("_B") or name == "l2_bytes":
                        v *= UNIT.get(u.get(k, "byte"), 1.0)
                    rec[name] = v
                except ValueError:
                    pass
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[k] or 0) for k in d
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                  and d[k] not in ("", "n/a")}
        tot = sum(stalls.values()) or 1.0
        rec["top_stalls"] = ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:3])
        yield rec


print("| kernel | grid x block | regs | us | DRAM rd+wr MB | SM % | mem % | occupancy % | tensor % | top stalls |")
print("|---|---|---|---|---|---|---|---|---|---|")
traffic = {}
for rep in sys.argv[1:]:
    for r in rows(rep):
        mb = (r.get("dram_read_B", 0) + r.get("dram_write_B", 0)) / 1e6
        print(f"| {r['kernel']} | {r.get('grid', 0):.0f} x {r.get('block', 0):.0f} | {r.get('regs', 0):.0f} | "
              f"{r.get('duration_us', 0):.1f} | {mb:.2f} | {r.get('sm_pct', 0):.1f} | {r.get('mem_pct', 0):.1f} | "
              f"{r.get('occupancy_pct', 0):.1f} | {r.get('tensor_pct', 0):.1f} | {r['top_stalls']} |")
        traffic.setdefault(r["kernel"], []).append(mb * 1e6)
sys.stderr.write(json.dumps({k: sum(v) / len(v) for k, v in traffic.items()}) + "\n")

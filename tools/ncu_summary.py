"""Summarise an ncu --set full report into markdown rows (and JSON) for profiles/.
    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--json out.json]"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex_%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts_%"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_%"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1_ld_sectors"),
]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
         "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
             .replace("(anonymous namespace)::", "").replace("sacd::", "").replace("unnamed>::", ""),
             "grid": vals[hdr.index("Grid Size")] if "Grid Size" in hdr else ""}
        for m, short in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if u in SCALE:
                    v *= SCALE[u]
                d[short] = v
        res.append(d)
    return res


def md(res):
    lines = ["| kernel | grid | time ms | DRAM GB (r+w) | DRAM % | L1TEX % | LTS % | L1 hit % | L2 hit % | occ % | issue % | regs |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for d in res:
        lines.append(f"| {d['kernel']} | {d['grid']} | {d.get('time', 0)*1e3:.3f} | "
                     f"{(d.get('dram_read', 0) + d.get('dram_write', 0))/1e9:.3f} | {d.get('dram_%', 0):.1f} | "
                     f"{d.get('l1tex_%', 0):.1f} | {d.get('lts_%', 0):.1f} | {d.get('l1_hit_%', 0):.1f} | "
                     f"{d.get('l2_hit_%', 0):.1f} | {d.get('occupancy_%', 0):.1f} | {d.get('issue_%', 0):.1f} | "
                     f"{int(d.get('regs', 0))} |")
    return "\n".join(lines)


if __name__ == "__main__":
    res = load(sys.argv[1])
    print(md(res))
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)

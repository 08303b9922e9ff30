"""Summarise an `ncu --set full --page raw --csv` export of MTTKRP launches into profiles/:
per launch the time, DRAM bytes, L1 / L2 hit rates and throughputs, occupancy, issue and the
L1 data-pipe wavefront utilisation; with --traffic, also rewrite profiles/traffic.json (the
mean DRAM bytes per launch that bench.py reports as roofline.traffic).
    python tools/ncu_mttkrp_summary.py gpurun_out/f2_mttkrp_full.csv profiles/r01_prof_mttkrp_c4_default.json --traffic"""
import csv
import json
import sys

SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
         "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}


def main():
    src, dst = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(line for line in open(src) if line.startswith('"')))
    hdr, units = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        def num(k):
            i = hdr.index(k)
            return float(v[i].replace(",", "")) * SCALE.get(units[i], 1.0)
        out.append(dict(
            kernel=v[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("sacd::", ""),
            grid=v[hdr.index("Grid Size")], time_s=num("gpu__time_duration.sum"),
            dram_read=num("dram__bytes_read.sum"), dram_write=num("dram__bytes_write.sum"),
            l1tex_pct=num("l1tex__throughput.avg.pct_of_peak_sustained_active"),
            lsu_wavefront_pct=num("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
            lts_pct=num("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            l1_hit_pct=num("l1tex__t_sector_hit_rate.pct"), l2_hit_pct=num("lts__t_sector_hit_rate.pct"),
            occupancy_pct=num("sm__warps_active.avg.pct_of_peak_sustained_active"),
            issue_pct=num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            regs=num("launch__registers_per_thread"), warp_inst=num("smsp__inst_executed.sum")))
    json.dump(out, open(dst, "w"), indent=1)
    for d in out:
        print({k: (round(x, 4) if isinstance(x, float) else x) for k, x in d.items()})
    if "--traffic" in sys.argv and out:
        tr = sum(d["dram_read"] + d["dram_write"] for d in out) / len(out)
        json.dump({"c4_R64_f64_mttkrp": tr,
                   "_about": f"dram__bytes_read.sum + dram__bytes_write.sum per default MTTKRP launch "
                             f"({out[0]['kernel']}), mean of the U/V/W launches of sweep 7 of c4 fp64 R=64, "
                             f"from {dst} (ncu --set full --clock-control none)"},
                  open("profiles/traffic.json", "w"), indent=1)
        print("traffic per launch", tr)


if __name__ == "__main__":
    main()

"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of bench.py: per
kernel class, launches, total and mean duration, and share of the libsacd kernel time.  The
per-launch times are serialised and cold-cache, so the SHARE is what is compared with the
bench's live kernel_ms_per_sweep, not the absolute.
    python tools/launch_summary.py gpurun_out/f1_launches.csv [--json out.json] [--csv trimmed.csv]"""
import collections
import csv
import json
import re
import sys

CLASSES = [("mttkrp", r"k_mttkrp"), ("fixup", r"k_fix[12]"), ("prepare", r"k_prepare"),
           ("rows", r"k_sacd_rows"), ("gram", r"k_gram_"), ("finalize", r"k_finalize"),
           ("pack", r"k_pack_rows|k_chunk_mask")]


def main():
    path = sys.argv[1]
    lines = [ln for ln in open(path) if ln.startswith('"')]  # skip ncu's ==PROF== / ==WARNING== lines
    rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
    ours = [r for r in rows if "sacd::" in r["Kernel Name"]]
    agg = collections.OrderedDict()
    for r in ours:
        name = r["Kernel Name"]
        cls = next((c for c, p in CLASSES if re.search(p, name)), "other")
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}[r["Metric Unit"]]
        t = float(r["Metric Value"].replace(",", "")) * scale
        a = agg.setdefault(cls, {"launches": 0, "ms": 0.0, "kernels": set()})
        a["launches"] += 1
        a["ms"] += t
        a["kernels"].add(re.sub(r"\(.*", "", name.replace("void ", "").replace("sacd::<unnamed>::", "")))
    tot = sum(a["ms"] for a in agg.values())
    out = {}
    print("| class | launches | total ms | mean ms | share |")
    print("|---|---|---|---|---|")
    for c, a in sorted(agg.items(), key=lambda kv: -kv[1]["ms"]):
        out[c] = {"launches": a["launches"], "total_ms": a["ms"], "mean_ms": a["ms"] / a["launches"],
                  "share": a["ms"] / tot, "kernels": sorted(a["kernels"])}
        print(f"| {c} | {a['launches']} | {a['ms']:.2f} | {a['ms'] / a['launches']:.4f} | {a['ms'] / tot:.3f} |")
    print(f"total libsacd kernel ms: {tot:.2f} over {len(ours)} launches (of {len(rows)} in the list)")
    if "--json" in sys.argv:
        json.dump({"source": path, "libsacd_launches": len(ours), "total_ms": tot, "classes": out},
                  open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
    if "--csv" in sys.argv:
        with open(sys.argv[sys.argv.index("--csv") + 1], "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["ID", "Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "unit"])
            for r in ours:
                w.writerow([r["ID"], re.sub(r"\(.*", "", r["Kernel Name"]), r["Grid Size"], r["Block Size"],
                            r["Metric Value"], r["Metric Unit"]])


if __name__ == "__main__":
    main()

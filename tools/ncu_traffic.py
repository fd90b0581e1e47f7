"""DRAM traffic per frame of every render kernel from an `ncu --set full`
capture of ONE whole frame:  python tools/ncu_traffic.py REP OUT.json [SUMMARY.txt]

Maps ncu kernel names to the names the ABI's kernel timeline uses (bench.py
kernels{}), sums launches of the same kernel, and writes
{name: dram_read + dram_write bytes}.  Optionally writes a text summary with
duration, DRAM bytes, achieved occupancy, issue utilisation and pipe shares."""
import csv
import io
import json
import re
import subprocess
import sys

MAP = [(r"preprocess_geo_kernel", "preprocess_geo"),
       (r"preprocess_color_kernel", "preprocess_color"),
       (r"depth_key32_kernel", "depth_key32"), (r"depth_fixup_kernel", "depth_fixup"),
       (r"radix_hist_kernel<unsigned int>", "radix32_hist"),
       (r"radix_plan_kernel<unsigned int>", "radix32_plan"),
       (r"onesweep_pass_kernel<unsigned int>", "radix32_pass"),
       (r"radix_hist_kernel<unsigned long long>", "radix64_hist"),
       (r"radix_plan_kernel<unsigned long long>", "radix64_plan"),
       (r"onesweep_pass_kernel<unsigned long long>", "radix64_pass"),
       (r"frame_start_kernel", "frame_start"),
       (r"color_ranked_kernel", "color_ranked"), (r"blend_kernel", "blend")]
for k in ["bin_gather", "row_scan", "bin_pairs", "seg_table", "seg_count", "seg_scan",
          "tile_scan", "seg_place", "bin_rows", "slice_plan", "slice_col_prefix",
          "slice_b_filter"]:
    MAP.append((k + "_kernel", k))

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
           "smsp__inst_executed.sum"]


def short(name):
    for pat, nm in MAP:
        if pat in name:
            return nm
    return name.split("(")[0]


def main(rep, out, summary=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    agg = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0,
             "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
    for r in rows[2:]:
        nm = short(r[hdr.index("Kernel Name")])
        a = agg.setdefault(nm, {m: 0.0 for m in METRICS} | {"launches": 0})
        a["launches"] += 1
        for m in METRICS:
            if m not in hdr:
                continue
            i = hdr.index(m)
            v = float(r[i].replace(",", "") or 0)
            a[m] += v * scale.get(units[i], 1.0) if m.startswith(("dram", "gpu__time")) else v
    traffic = {nm: int(a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]) for nm, a in agg.items()}
    with open(out, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    if summary:
        tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
        with open(summary, "w") as f:
            f.write(f"ncu --set full, one config-3 frame (3M Gaussians, SH3, 1920x1080), "
                    f"{sum(a['launches'] for a in agg.values())} launches, {tot:.1f} us "
                    f"(serialised, cold)\n")
            f.write(f"{'kernel':18s} {'n':>2s} {'us':>8s} {'share':>6s} {'DRAM MB':>8s} "
                    f"{'GB/s':>7s} {'warps%':>6s} {'sm%':>5s} {'fp64%':>6s} {'fma%':>5s} "
                    f"{'alu%':>5s}\n")
            for nm, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
                n = a["launches"]
                us = a["gpu__time_duration.sum"]
                mb = (a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]) / 1e6
                f.write(f"{nm:18s} {n:2d} {us:8.1f} {100 * us / tot:5.1f}% {mb:8.1f} "
                        f"{mb / 1e3 / (us * 1e-6) if us else 0:7.0f} "
                        f"{a['sm__warps_active.avg.pct_of_peak_sustained_active'] / n:6.1f} "
                        f"{a['sm__throughput.avg.pct_of_peak_sustained_elapsed'] / n:5.1f} "
                        f"{a['sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'] / n:6.1f} "
                        f"{a['sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'] / n:5.1f} "
                        f"{a['sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active'] / n:5.1f}\n")
    print(json.dumps(traffic))


if __name__ == "__main__":
    main(*sys.argv[1:])

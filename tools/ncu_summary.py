"""Key metrics per kernel + top stall lines from an .ncu-rep (run in the build container)."""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
           "smsp__inst_executed.sum", "launch__grid_size",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
           "smsp__thread_inst_executed_per_inst_executed.ratio"]


def ncu(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main(rep, top=12, only=None):
    rows = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    for k, r in enumerate(rows[2:]):
        name = r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1]
        if only is not None and k not in only:
            continue
        print(f"=== [{k}] {name}")
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"  {m:66s} {r[i]:>16s} {units[i]}")
        if only is not None and k not in only:
            continue
        try:
            src = ncu([rep, "--page", "source", "--csv", "--launch-skip", str(k),
                       "--launch-count", "1"])
        except Exception as e:  # noqa: BLE001
            print(f"    (source page unavailable: {e})")
            continue
        srows = list(csv.reader(io.StringIO(src)))
        if len(srows) < 3:
            continue
        sh = srows[1]
        si, so = sh.index("Warp Stall Sampling (All Samples)"), sh.index("Source")
        def num(x):
            try:
                return float(x[si] or 0)
            except (ValueError, IndexError):
                return 0.0
        body = [x for x in srows[2:] if len(x) > max(si, so)]
        tot = sum(num(x) for x in body) or 1.0
        for x in sorted(body, key=lambda x: -num(x))[:top]:
            print(f"    {100 * num(x) / tot:5.1f}%  {x[so][:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12,
         {int(x) for x in sys.argv[3].split(",")} if len(sys.argv) > 3 else None)

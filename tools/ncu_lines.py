"""Per-CUDA-source-line stall samples and executed instructions of one kernel
in an .ncu-rep:  python tools/ncu_lines.py REP LAUNCH_INDEX [TOP]"""
import csv
import io
import subprocess
import sys


def main(rep, k, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass", "--launch-skip", str(k), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    fname, rows = "?", []
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or r[0] == "":
            continue
        try:
            rows.append((fname, int(r[0]), r[1], float(r[4] or 0), float(r[7] or 0)))
        except (ValueError, IndexError):
            pass
    ts = sum(x[3] for x in rows) or 1
    ti = sum(x[4] for x in rows) or 1
    print(f"total stall samples {ts:.0f}, warp instructions {ti:.0f}")
    for f, ln, src, s, i in sorted(rows, key=lambda x: -x[3])[:top]:
        print(f"{100 * s / ts:5.1f}% stall {100 * i / ti:5.1f}% inst  {f}:{ln:<4} {src.strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 30)

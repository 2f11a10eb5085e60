"""Per-source-line stall samples and executed instructions of one kernel in an
ncu report (dev tool).

    python tools/ncu_lines_src.py report.ncu-rep [top]

Uses `ncu --page source --print-source cuda,sass` (the build has -lineinfo);
prints the source lines with the most warp-stall samples and their top
stall reasons."""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    idx = {h: i for i, h in enumerate(hdr)}
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    lines = []
    total = 0
    for r in rows:
        if not r or not r[0].isdigit() or len(r) < len(hdr):
            continue
        try:
            s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:  # a source line the CSV export split oddly
            continue
        total += s
        reasons = sorted(((int(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
        lines.append((s, int(r[0]), r[1].strip()[:70], int(r[idx["Instructions Executed"]] or 0),
                      reasons))
    lines.sort(reverse=True)
    print(f"total samples {total}")
    for s, ln, src, ins, rs in lines[:top]:
        rtxt = ", ".join(f"{n} {v}" for v, n in rs if v)
        print(f"{100.0 * s / max(total, 1):5.1f}%  L{ln:<4} inst {ins:>10}  {src:<70} | {rtxt}")


if __name__ == "__main__":
    main()

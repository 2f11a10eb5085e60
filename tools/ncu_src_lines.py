"""Per-source-line warp-stall samples and executed instructions of one kernel,
over every source file it inlines (dev tool; the build has -lineinfo).

    python tools/ncu_src_lines.py report.ncu-rep <kernel-regex> [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", "regex:" + kern], capture_output=True, text=True).stdout
    cur, res = None, []
    for r in csv.reader(io.StringIO(out)):
        if len(r) >= 2 and r[0] in ("File Path", "File Name"):
            cur = r[1].split("/")[-1]
            continue
        if not r or not r[0].isdigit() or len(r) < 8:
            continue
        try:
            s, ins = int(r[4] or 0), int(r[7] or 0)
        except ValueError:
            continue
        res.append((cur, int(r[0]), s, ins, r[1].strip()[:80]))
    S = sum(x[2] for x in res) or 1
    I = sum(x[3] for x in res) or 1
    print(f"stall samples {S}, warp instructions {I}")
    for f, ln, s, ins, src in sorted(res, key=lambda x: -x[2])[:top]:
        print(f"{100 * s / S:5.1f}% stalls {100 * ins / I:5.1f}% inst  {f}:{ln:<4} {src}")


if __name__ == "__main__":
    main()

"""Attribute ncu SASS-level stall samples / executed instructions to source lines.

    python tools/ncu_lines.py <obj.o> <kernel-substring> <report.ncu-rep> [top]

Extracts the cubin from the object, disassembles it with line info
(nvdisasm -g), exports the report's source page (SASS view) and sums
"Warp Stall Sampling (All Samples)" and "Instructions Executed" per source
line of the innermost (possibly inlined) location.  Dev tool.
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile


def main():
    obj, kname, rep = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True,
                   capture_output=True)
    cub = glob.glob(os.path.join(tmp, "*.cubin"))[0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    # split per function, keep the one matching kname
    addr2line, cur, infn = {}, None, False
    for line in dis.split("\n"):
        if line.startswith("//--------------------- .text."):
            infn = kname in line
            continue
        if not infn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m2 = re.search(r"/\*([0-9a-f]{4,})\*/", line)
        if m2 and cur is not None:
            addr2line[int(m2.group(1), 16)] = cur
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isamp, iex = (hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"),
                      hdr.index("Instructions Executed"))
    samp, ex, tot = collections.Counter(), collections.Counter(), 0.0
    base = None
    for r in rows[2:]:
        try:
            a = int(r[ia], 16)
        except (ValueError, IndexError):
            continue
        if base is None:
            base = a  # the report holds absolute addresses; the first row is offset 0
        a -= base
        ln = addr2line.get(a, ("?", 0))
        s = float(r[isamp] or 0)
        samp[ln] += s
        ex[ln] += float(r[iex] or 0)
        tot += s
    srcs = {}
    for (f, ln), s in samp.most_common(top):
        if f not in srcs:
            p = glob.glob(os.path.join(os.path.dirname(__file__), "..", "**", f), recursive=True)
            srcs[f] = open(p[0]).read().split("\n") if p else []
        text = srcs[f][ln - 1].strip()[:70] if 0 < ln <= len(srcs[f]) else ""
        print(f"{f}:{ln:<5d} {100 * s / max(tot, 1):5.1f}%  ex={ex[(f, ln)] / 1e6:8.2f}M  {text}")


if __name__ == "__main__":
    main()

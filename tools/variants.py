"""Build compile-time variants of the CUDA library for A/B timing (dev tool).

    python tools/variants.py name1:-DFOO=1,-DBAR=2 name2:-DFOO=2 ...

Each variant goes to build/var/<name>/libisinglink_b200.so; select one at
run time with ISINGLINK_B200_LIB=<path>.
"""
import glob
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_01579_b200 import build as b  # noqa: E402


def main():
    procs = []
    for spec in sys.argv[1:]:
        name, _, flags = spec.partition(":")
        flags = [f for f in flags.split(",") if f]
        out = os.path.join(b.ROOT, "build", "var", name)
        os.makedirs(out, exist_ok=True)
        objs = []
        for src in sorted(glob.glob(os.path.join(b.CSRC, "*.cu"))):
            obj = os.path.join(out, os.path.basename(src)[:-3] + ".o")
            objs.append(obj)
            procs.append((src, subprocess.Popen([b.nvcc(), *b.ARCH, *b.NVCC_FLAGS, *flags, "-c",
                                                 src, "-o", obj])))
        procs.append(("link", (out, objs)))
    pending = []
    for src, p in procs:
        if src == "link":
            pending.append(p)
            continue
        if p.wait() != 0:
            raise SystemExit(f"nvcc failed on {src}")
    for out, objs in pending:
        subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-o", os.path.join(out, "libisinglink_b200.so"),
                        *objs, "-cudart", "static"], check=True)
        print(os.path.join(out, "libisinglink_b200.so"))


if __name__ == "__main__":
    main()

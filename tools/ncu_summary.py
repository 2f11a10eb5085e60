"""Summarise an ncu report for profiles/ (dev tool).

    python tools/ncu_summary.py report.ncu-rep > profiles/<name>.txt

Per kernel: duration, registers, occupancy, pipe utilisation, DRAM bytes,
issue-stall breakdown (pc sampling) and the SOL / scheduler sections.
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for v in rows[2:]:
        d = dict(zip(hdr, v))
        u = dict(zip(hdr, units))
        print(f"== {d.get('Kernel Name', '?')[:110]}")
        for k in KEYS:
            if k in d:
                print(f"   {k:70s} {d[k]} {u.get(k, '')}")
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(x or 0)
              for k, x in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        tot = sum(st.values()) or 1.0
        print("   issue-stall samples (%):", ", ".join(
            f"{k} {100 * x / tot:.1f}" for k, x in sorted(st.items(), key=lambda z: -z[1])[:10]))
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    for r in csv.reader(io.StringIO(det)):
        if len(r) > 14 and r[-4] in ("GPU Speed Of Light Throughput", "Occupancy",
                                     "Scheduler Statistics", "Warp State Statistics"):
            print(f"   [{r[-4]}] {r[-3]}: {r[-1]} {r[-2]}")


if __name__ == "__main__":
    main()

#!/bin/bash
# Round-end measurement recipe (run under gpurun from the repo root):
#   bench line, reference arm, ncu launch list of the bench command and one
#   --set full capture of the dominant kernel.  Outputs land in gpurun_out/.
set -u
TAG=${1:-r01}
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_launches.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_anneal_fast -c 1 \
    -o gpurun_out/${TAG}_anneal_full python tools/quick_bench.py 16 16 45864 fp32 1 \
    > gpurun_out/${TAG}_anneal_full.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_front -c 1 \
    -o gpurun_out/${TAG}_front_full python tools/quick_bench.py 16 16 45864 fp32 1 \
    > gpurun_out/${TAG}_front_full.log 2>&1
tail -c 600 gpurun_out/${TAG}_bench.json

# one ncu --set full capture each of the front end and the anneal (16x16 slot)
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_front_rows|k_anneal_fast' -c 2 -o gpurun_out/full_r02 python tools/quick_bench.py 16 16 45864 fp32 1 > gpurun_out/prof_full.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/prof_full.log

# round check: -m gpu suite, smoke, bench (device + e2e), reference arm, ncu launch list, ncu --set full of the top kernels
cd $GRAFT_REPO_ROOT
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -q -s --tb=short -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-other-configs > gpurun_out/b_ncu.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_front_rows|k_anneal_fast|k_select_decode' -c 3 -o gpurun_out/full_round python tools/quick_bench.py 16 16 45864 fp32 1 > gpurun_out/prof_full.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/gputests.log
cat gpurun_out/smoke.log | tail -2
cat gpurun_out/bench.json

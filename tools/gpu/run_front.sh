# front-end change check: parity tests touching the front end + bench (no CPU legs)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_slot_gpu.py tests/test_api_gpu.py tests/test_baseline_curves.py tests/test_multi_gpu.py -m gpu -q -s --tb=short -p no:cacheprovider > gpurun_out/front_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/front_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-other-configs > gpurun_out/bench_front.json 2> gpurun_out/bench_front.err; echo "bench rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_front_rows -c 1 -o gpurun_out/front_r02 python tools/quick_bench.py 16 16 45864 fp32 1 > gpurun_out/front_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/front_tests.log

# quick GPU check: selected tests + bench + reference arm
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_reference_suite_gpu.py tests/test_gpu_parity.py -m gpu -q -s --tb=short -p no:cacheprovider > gpurun_out/quick_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quick_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
tail -3 gpurun_out/quick_tests.log

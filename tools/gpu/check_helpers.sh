cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_helpers_gpu.py tests/test_api_gpu.py tests/test_reference_suite_gpu.py tests/test_padding_counts_gpu.py tests/test_gpu_parity.py -m gpu -q --tb=short -p no:cacheprovider 2>&1 | tail -15

# the reference's acceptance suite (pkg/tests/test_acceptance.py) with the CUDA kernel active
cd $GRAFT_REPO_ROOT/oracle/_ref/pkg_tests
export PYTHONPATH=$GRAFT_REPO_ROOT/tests:$GRAFT_REPO_ROOT
export ISINGLINK_REF_ACTIVATE=1
timeout 2400 python -m pytest -s -v -p ref_suite_plugin -p no:cacheprovider -c /dev/null --rootdir . test_acceptance.py -k "not criterion_08" > $GRAFT_REPO_ROOT/gpurun_out/ref_acceptance.log 2>&1
echo "rc=$?"
grep -E "ACCEPTANCE|passed|failed|reference package" $GRAFT_REPO_ROOT/gpurun_out/ref_acceptance.log

# A/B of library variants on the small register layouts NT <= 3 (dev tool,
# run under gpurun): bit-identity against build/var/old, then slot timings.
cd $GRAFT_REPO_ROOT
ISINGLINK_B200_LIB=build/var/old/libisinglink_b200.so python tools/dump_outputs.py gpurun_out/ab_old.npz 2>&1 | grep -v Warn
for v in "$@"; do
  echo "[$v]"; ISINGLINK_B200_LIB=build/var/$v/libisinglink_b200.so python tools/dump_outputs.py gpurun_out/ab_$v.npz gpurun_out/ab_old.npz 2>&1 | grep -v Warn
done
for rep in 1 2; do
for v in "$@"; do
  L=build/var/$v/libisinglink_b200.so
  for shape in "8 16 45864 fp32 5" "8 16 45864 fp32 5 8" "6 16 45864 fp32 5" "12 16 45864 fp32 3" "16 16 45864 fp32 3"; do
    ISINGLINK_B200_LIB=$L python tools/quick_bench.py $shape 2>&1 | grep -v Warn | tail -1 | sed "s/^/[$v] /"
  done
  ISINGLINK_B200_LIB=$L python tools/vpp_time.py 2>&1 | grep -v Warn | head -1 | sed "s/^/[$v] vpp /"
done
done

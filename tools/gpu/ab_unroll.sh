# A/B of the step-loop unroll factor (dev tool, run under gpurun): bit-identity
# of the detect outputs of build/var/<v> against build/var/old, then slot
# timings on the BASELINE shapes.  Variants: $@
cd $GRAFT_REPO_ROOT
ISINGLINK_B200_LIB=build/var/old/libisinglink_b200.so python tools/dump_outputs.py gpurun_out/ab_old.npz 2>&1 | grep -v Warn
for v in "$@"; do
  echo "[$v]"; ISINGLINK_B200_LIB=build/var/$v/libisinglink_b200.so python tools/dump_outputs.py gpurun_out/ab_$v.npz gpurun_out/ab_old.npz 2>&1 | grep -v Warn
done
for rep in 1 2; do
for v in old "$@"; do
  L=build/var/$v/libisinglink_b200.so
  for shape in "16 16 45864 fp32 5" "8 16 45864 fp32 5" "16 64 45864 fp32 3 8" "16 64 45864 fp32 3 128" "12 16 45864 fp32 3" "16 16 45864 mixed 5"; do
    ISINGLINK_B200_LIB=$L python tools/quick_bench.py $shape 2>&1 | grep -v Warn | tail -1 | sed "s/^/[$v] /"
  done
done
done

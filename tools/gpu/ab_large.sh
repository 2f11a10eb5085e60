# large-shape slot timings (n_t = 28, 32, 26) for the default build and each named variant (build/var/<v>)
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for v in default "$@"; do
  if [ "$v" = default ]; then L=paper_2510_01579_b200/_lib/libisinglink_b200.so; else L=build/var/$v/libisinglink_b200.so; fi
  for nt in 28 32 26; do ISINGLINK_B200_LIB=$L python tools/quick_bench.py $nt 16 45864 fp32 3 2>&1 | grep -v Warn | tail -1 | sed "s/^/[$v] /"; done
done; done

# A/B of library variants (dev tool, run under gpurun): bit-identity of the
# detect outputs against build/var/old, then slot timings.  Variants: $@
set -u
python tools/dump_outputs.py gpurun_out/ab_new.npz 2>&1 | grep -v Warn
ISINGLINK_B200_LIB=build/var/old/libisinglink_b200.so python tools/dump_outputs.py gpurun_out/ab_old.npz 2>&1 | grep -v Warn
python -c "
import numpy as np
a=np.load('gpurun_out/ab_new.npz'); b=np.load('gpurun_out/ab_old.npz')
bad=[k for k in a if not np.array_equal(a[k],b[k],equal_nan=True)]
print('bit-identical' if not bad else 'DIFF: '+' '.join(bad))
"
for v in old "$@"; do ISINGLINK_B200_LIB=build/var/$v/libisinglink_b200.so python tools/quick_bench.py 16 16 45864 fp32 5 2>&1 | grep -v Warn; done
python tools/quick_bench.py 16 16 45864 fp32 5 2>&1 | grep -v Warn
ISINGLINK_B200_LIB=build/var/old/libisinglink_b200.so python tools/quick_bench.py 8 16 45864 fp32 3 2>&1 | grep -v Warn
python tools/quick_bench.py 8 16 45864 fp32 3 2>&1 | grep -v Warn
python tools/quick_bench.py 16 64 45864 fp32 3 2>&1 | grep -v Warn
ISINGLINK_B200_LIB=build/var/old/libisinglink_b200.so python tools/quick_bench.py 16 64 45864 fp32 3 2>&1 | grep -v Warn
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3

# finish fused into the PFHX pole kernel (last block per item tile) vs the finish kernel
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s4s_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/s4s_pytest_gpu.log; tail -1 gpurun_out/checked_run.log
for v in 1 0; do REXI_FUSE_FINISH=$v python tests/scripts/staging_identity.py gpurun_out/s4s_f$v.npz; done
python -c "
import numpy as np
a=np.load('gpurun_out/s4s_f1.npz'); b=np.load('gpurun_out/s4s_f0.npz')
print('fused finish bit-identical:', all(np.array_equal(a[k], b[k]) for k in a.files), len(a.files))"
for v in 1 0 1 0; do REXI_FUSE_FINISH=$v python bench.py --steps 300 --no-cpu-baseline > gpurun_out/s4s_b$v.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/s4s_b$v.json'));print('fuse=$v', d['ms_per_step'], d['roofline']['kernel_ms_avg'], d['gpu_launches'])"; done
for v in 1 0; do REXI_FUSE_FINISH=$v python bench.py --config c3 --steps 200 --no-cpu-baseline > gpurun_out/s4s_c3_b$v.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/s4s_c3_b$v.json'));print('c3 fuse=$v', d['ms_per_step'], d['roofline']['kernel_ms_avg'])"; done
for v in 1 0; do REXI_FUSE_FINISH=$v python tools/time_partial.py c2 200 | tail -1; done

# A/B of pole-kernel staging modes (REXI_R2X_BULK=0 register-staged copy, 1 bulk copy, 2 bulk + batched denominators)
set -x
mkdir -p gpurun_out
timeout 600 env REXI_R2X_BULK=2 python -m pytest tests/test_gpu_parity.py -q -x -k "r2x or pfhx or c2 or full_grid" > gpurun_out/s4f_pytest.log 2>&1; echo pytest_rc=$?
tail -1 gpurun_out/s4f_pytest.log
for b in 1 2 1 2; do REXI_R2X_BULK=$b python bench.py --steps 200 --no-cpu-baseline > gpurun_out/s4f_bench_b$b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/s4f_bench_b$b.json'));print('bulk=$b', d['ms_per_step'], d['roofline']['kernel_ms_avg'], d['roofline']['frac'], d['roofline']['fp64_pipe_frac'])"; done
for b in 1 2; do REXI_R2X_BULK=$b python tools/time_partial.py c2 200 | tail -1; done

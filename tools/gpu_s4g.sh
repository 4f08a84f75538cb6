# persistent PFHX kernel (REXI_R2X_BULK=2) vs the bulk-staged one: parity + A/B timing
set -x
mkdir -p gpurun_out
timeout 900 env REXI_R2X_BULK=2 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partial.py tests/test_gpu_checked.py -q -x > gpurun_out/s4g_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/s4g_pytest.log
for b in 1 2; do REXI_R2X_BULK=$b python tools/time_pole_counts.py; done
for b in 1 2 1 2; do REXI_R2X_BULK=$b python bench.py --steps 200 --no-cpu-baseline > gpurun_out/s4g_bench_b$b.json 2>gpurun_out/s4g_bench_b$b.err; python -c "import json;d=json.load(open('gpurun_out/s4g_bench_b$b.json'));print('bulk=$b', d['ms_per_step'], d['roofline']['kernel_ms_avg'], d['roofline']['frac'], d['roofline']['fp64_pipe_frac'])"; done

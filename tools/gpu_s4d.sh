# bulk-copy pole-table staging (pole_kernel_r2x_bulk) vs the register-staged copy: parity + A/B timing
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partial.py -q -x > gpurun_out/s4d_pytest.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/s4d_pytest.log
for b in 0 1 0 1; do REXI_R2X_BULK=$b python bench.py --steps 200 --no-cpu-baseline > gpurun_out/s4d_bench_b$b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/s4d_bench_b$b.json'));print('bulk=$b', d['ms_per_step'], d['roofline']['kernel_ms_avg'], d['roofline']['frac'])"; done
for b in 0 1; do REXI_R2X_BULK=$b python tools/time_partial.py c2 200 > gpurun_out/s4d_partial_b$b.jsonl; cat gpurun_out/s4d_partial_b$b.jsonl; done
for b in 0 1; do REXI_R2X_BULK=$b python tools/time_partial.py c3 100 > gpurun_out/s4d_partial_c3_b$b.jsonl; cat gpurun_out/s4d_partial_c3_b$b.jsonl; done

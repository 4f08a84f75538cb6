set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py -q -x > gpurun_out/pytest_fused_r02e.log 2>&1; echo fused_rc=$?
tail -30 gpurun_out/pytest_fused_r02e.log
timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c1_r02e.json 2> gpurun_out/bench_c1_r02e.err; cat gpurun_out/bench_c1_r02e.json; tail -3 gpurun_out/bench_c1_r02e.err
timeout 1200 python -m pytest tests/test_gpu_checked.py -q -x > gpurun_out/pytest_checked_r02e.log 2>&1; echo checked_rc=$?
tail -30 gpurun_out/pytest_checked_r02e.log; tail -20 gpurun_out/checked_run.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r02e.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_r02e.log

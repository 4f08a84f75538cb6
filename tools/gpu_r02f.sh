set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_checked.py -q -x > gpurun_out/pytest_fused_r02f.log 2>&1; echo fused_rc=$?
tail -5 gpurun_out/pytest_fused_r02f.log; tail -5 gpurun_out/checked_run.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_small -s 5 -c 1 -o gpurun_out/r02f_small python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_ncu.log 2>&1; echo ncu_rc=$?
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r02f.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_r02f.log

set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_checked.py -q -x > gpurun_out/pytest_fused_r02h.log 2>&1; echo fused_rc=$?
tail -30 gpurun_out/pytest_fused_r02h.log; grep -v ": ok" gpurun_out/checked_run.log | tail -5
timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c1_r02h.json 2> gpurun_out/bench_c1_r02h.err; cat gpurun_out/bench_c1_r02h.json; tail -3 gpurun_out/bench_c1_r02h.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_small -s 5 -c 1 -o gpurun_out/r02h_small python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02h_ncu.log 2>&1; echo ncu_rc=$?

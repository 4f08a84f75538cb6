set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_checked.py -q -x > gpurun_out/pytest_fused_r02k.log 2>&1; echo fused_rc=$?
tail -3 gpurun_out/pytest_fused_r02k.log; grep -v ": ok" gpurun_out/checked_run.log | tail -3
timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c1_r02k.json 2> gpurun_out/bench_c1_r02k.err; tail -3 gpurun_out/bench_c1_r02k.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_small -s 5 -c 1 -o gpurun_out/r02k_small python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02k_ncu.log 2>&1; echo ncu_rc=$?
MASTER_ADDR=127.0.0.1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --backend gloo --steps 5 --warmup 3 --config c2 > gpurun_out/bench_gloo2_r02k.json 2> gpurun_out/bench_gloo2_r02k.err; echo gloo_rc=$?; tail -3 gpurun_out/bench_gloo2_r02k.err

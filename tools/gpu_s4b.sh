# NCCL code path on the box's one GPU: world-size-1 process group (test + bench --dist under torchrun)
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_distributed.py -q > gpurun_out/s4b_pytest_dist.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/s4b_pytest_dist.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --dist --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/s4b_bench_c2_nccl1.json 2> gpurun_out/s4b_bench_c2_nccl1.err; echo dist_rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --dist --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s4b_bench_c4_nccl1.json 2> gpurun_out/s4b_bench_c4_nccl1.err; echo dist4_rc=$?
cut -c1-300 gpurun_out/s4b_bench_c2_nccl1.json; grep -o '"ranks.*' gpurun_out/s4b_bench_c2_nccl1.json
grep -i "nccl" gpurun_out/s4b_bench_c2_nccl1.err | head -20

set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r02b.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_r02b.log
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c2_r02b.json 2> gpurun_out/bench_c2_r02b.err; cat gpurun_out/bench_c2_r02b.json
python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_r02b.json 2> gpurun_out/bench_c4_r02b.err; cat gpurun_out/bench_c4_r02b.json
bash tools/gpu_profile.sh r02b
ls -la gpurun_out

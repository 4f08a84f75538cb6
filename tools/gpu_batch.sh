set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r02a.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_r02a.log
python tools/tune.py c2 pfhx,pfhr > gpurun_out/tune_c2_r02a.jsonl 2>&1
cat gpurun_out/tune_c2_r02a.jsonl
python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2_r02a.json 2> gpurun_out/bench_c2_r02a.err; cat gpurun_out/bench_c2_r02a.json

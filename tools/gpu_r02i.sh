set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r02i.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_r02i.log; grep -v ": ok" gpurun_out/checked_run.log | tail -3
for c in c1 c3; do timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_${c}_r02i.json 2> gpurun_out/bench_${c}_r02i.err; cat gpurun_out/bench_${c}_r02i.json | cut -c1-400; done
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c2_r02i.json 2> gpurun_out/bench_c2_r02i.err; cat gpurun_out/bench_c2_r02i.json | cut -c1-400

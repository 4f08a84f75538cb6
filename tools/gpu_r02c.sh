set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r02c.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_r02c.log
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c2_r02c.json 2> gpurun_out/bench_c2_r02c.err; cat gpurun_out/bench_c2_r02c.json; tail -3 gpurun_out/bench_c2_r02c.err
timeout 900 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize_run.py > gpurun_out/sanitize_memcheck_r02c.log 2>&1; echo memcheck_rc=$?
tail -5 gpurun_out/sanitize_memcheck_r02c.log
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_run.py > gpurun_out/sanitize_racecheck_r02c.log 2>&1; echo racecheck_rc=$?
tail -5 gpurun_out/sanitize_racecheck_r02c.log
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_run.py > gpurun_out/sanitize_synccheck_r02c.log 2>&1; echo synccheck_rc=$?
tail -5 gpurun_out/sanitize_synccheck_r02c.log

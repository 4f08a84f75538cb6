# Session-4 validation of HEAD (run under gpurun): GPU suite, smoke, C1/C2 bench lines.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s4a_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/s4a_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4a_smoke.log 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/s4a_smoke.log
python bench.py > gpurun_out/s4a_bench_c2.json 2> gpurun_out/s4a_bench_c2.err; echo c2_rc=$?
python bench.py --config c1 --no-cpu-baseline > gpurun_out/s4a_bench_c1.json 2> gpurun_out/s4a_bench_c1.err; echo c1_rc=$?
cut -c1-400 gpurun_out/s4a_bench_c2.json gpurun_out/s4a_bench_c1.json

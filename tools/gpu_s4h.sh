# Session-4 validation of the bulk-staged default: GPU suite, smoke, bench lines C1..C4, reference arm
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s4h_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/s4h_pytest_gpu.log; tail -1 gpurun_out/checked_run.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4h_smoke.log 2>&1; echo smoke_rc=$?
python bench.py > gpurun_out/s4h_bench_c2.json 2> gpurun_out/s4h_bench_c2.err; echo c2_rc=$?
python bench.py --config c1 --no-cpu-baseline > gpurun_out/s4h_bench_c1.json 2> gpurun_out/s4h_bench_c1.err; echo c1_rc=$?
python bench.py --config c3 --no-cpu-baseline > gpurun_out/s4h_bench_c3.json 2> gpurun_out/s4h_bench_c3.err; echo c3_rc=$?
python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s4h_bench_c4.json 2> gpurun_out/s4h_bench_c4.err; echo c4_rc=$?
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/s4h_ref_c2.json 2> gpurun_out/s4h_ref_c2.err; echo ref_rc=$?
python tools/time_partial.py c4 3 > gpurun_out/s4h_partial_c4.jsonl 2>&1
for c in c1 c2 c3 c4; do python -c "import json;d=json.load(open('gpurun_out/s4h_bench_$c.json'));print('$c', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['fp64_pipe_frac'], d['e2e']['value'], d['clocks'])"; done

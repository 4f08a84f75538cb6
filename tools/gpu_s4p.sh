# HEAD check: GPU suite, smoke, default bench line
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s4p_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/s4p_pytest_gpu.log; tail -1 gpurun_out/checked_run.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4p_smoke.log 2>&1; echo smoke_rc=$?; cat gpurun_out/s4p_smoke.log | tail -2
python bench.py > gpurun_out/s4p_bench_c2.json 2> gpurun_out/s4p_bench_c2.err; echo c2_rc=$?
python -c "import json;d=json.load(open('gpurun_out/s4p_bench_c2.json'));print(d['ms_per_step'], d['value'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['fp64_pipe_frac'], d['e2e']['value'], d['gpu_launches'], d['clocks'])"

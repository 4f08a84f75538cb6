# PFHX state without eta0 (hn eta0 = (n/mu) E): 162 registers, 3 blocks per SM: parity + timing
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s4k_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/s4k_pytest_gpu.log; tail -1 gpurun_out/checked_run.log
for i in 1 2; do python bench.py --steps 200 --no-cpu-baseline > gpurun_out/s4k_bench_c2_$i.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/s4k_bench_c2_$i.json'));print('c2', d['ms_per_step'], d['value'], d['roofline']['kernel_ms_avg'], d['roofline']['frac'], d['roofline']['fp64_pipe_frac'])"; done
for t in 8,8,3 8,4,2 8,2,2; do python bench.py --steps 100 --no-cpu-baseline --tuning $t > gpurun_out/s4k_bench_c2_t$t.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/s4k_bench_c2_t$t.json'));print('c2 tuning $t', d['ms_per_step'], d['roofline']['kernel_ms_avg'], d['roofline']['fp64_pipe_frac'])"; done
python bench.py --config c1 --no-cpu-baseline > gpurun_out/s4k_bench_c1.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/s4k_bench_c1.json'));print('c1', d['ms_per_step'], d['value'])"
python tools/time_partial.py c3 100 > gpurun_out/s4k_partial_c3.jsonl; head -1 gpurun_out/s4k_partial_c3.jsonl

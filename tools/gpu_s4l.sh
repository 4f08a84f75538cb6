# Validation of the shared-RHS PFHX default: GPU suite, smoke, bench C1..C4, reference arm, C2/C4 ncu, C4 ten steps, per-rank shares
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s4l_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/s4l_pytest_gpu.log; tail -1 gpurun_out/checked_run.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4l_smoke.log 2>&1; echo smoke_rc=$?
python bench.py > gpurun_out/s4l_bench_c2.json 2> gpurun_out/s4l_bench_c2.err; echo c2_rc=$?
python bench.py --config c1 --no-cpu-baseline > gpurun_out/s4l_bench_c1.json 2> gpurun_out/s4l_bench_c1.err; echo c1_rc=$?
python bench.py --config c3 --no-cpu-baseline > gpurun_out/s4l_bench_c3.json 2> gpurun_out/s4l_bench_c3.err; echo c3_rc=$?
python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s4l_bench_c4.json 2> gpurun_out/s4l_bench_c4.err; echo c4_rc=$?
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/s4l_ref_c2.json 2> gpurun_out/s4l_ref_c2.err; echo ref_rc=$?
for c in c1 c2 c3 c4; do python -c "import json;d=json.load(open('gpurun_out/s4l_bench_$c.json'));print('$c', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['fp64_pipe_frac'], d['e2e']['value'], d['clocks'])"; done
for c in c2 c3; do python tools/time_partial.py $c 200 > gpurun_out/s4l_partial_$c.jsonl 2>&1; done
python tools/time_partial.py c4 3 > gpurun_out/s4l_partial_c4.jsonl 2>&1
cat gpurun_out/s4l_partial_c*.jsonl
python examples/lrsw_gaussian.py 4096 1.0 10 > gpurun_out/s4l_c4_multistep10.txt 2>&1; cat gpurun_out/s4l_c4_multistep10.txt
bash tools/gpu_profile.sh s4l_c2
timeout 1200 ncu --set full --clock-control none -k regex:pole_kernel -c 1 -o gpurun_out/s4l_c4_pole python tools/prof_apply.py c4 1 > gpurun_out/s4l_ncu_c4.log 2>&1; echo ncu_c4=$?

set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r02q.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_r02q.log; grep -v ": ok" gpurun_out/checked_run.log | tail -3
for c in c4; do timeout 900 ncu --set full --clock-control none -k regex:"fft_|finish_kernel" -c 5 -o gpurun_out/r02q_aux_$c python tools/prof_apply.py $c 1 > gpurun_out/r02q_aux_$c.log 2>&1; echo ncu_$c=$?; done
timeout 900 ncu --set full --clock-control none -k regex:"fft_|finish_kernel" -c 5 -o gpurun_out/r02q_aux_c3 python tools/prof_apply.py c3 1 > gpurun_out/r02q_aux_c3.log 2>&1
for c in c3 c2; do timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_${c}_r02q.json 2> gpurun_out/bench_${c}_r02q.err; done

set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r02p.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_r02p.log
for c in c3 c4; do timeout 900 ncu --set full --clock-control none -k regex:"fft_|finish_kernel" -c 5 -o gpurun_out/r02p_aux_$c python tools/prof_apply.py $c 1 > gpurun_out/r02p_aux_$c.log 2>&1; echo ncu_$c=$?; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/r02p_c3_launches.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02p_c3_ncu1.log 2>&1
for c in c3 c2; do timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_${c}_r02p.json 2> gpurun_out/bench_${c}_r02p.err; done

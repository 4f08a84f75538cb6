set -x
mkdir -p gpurun_out
for c in c3 c4; do timeout 900 ncu --set full --clock-control none -k regex:"fft_|finish_kernel" -c 5 -o gpurun_out/r02v_aux_$c python tools/prof_apply.py $c 1 > gpurun_out/r02v_aux_$c.log 2>&1; echo ncu_$c=$?; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_small2 -s 5 -c 1 -o gpurun_out/r02v_small python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02v_ncu_small.log 2>&1; echo ncu_small=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02v_c2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02v_c2_ncu1.log 2>&1; echo ncu_c2=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02v_c3_launches.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02v_c3_ncu1.log 2>&1; echo ncu_c3=$?
for c in c3 c4; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_r02v.json 2> gpurun_out/bench_${c}_r02v.err; done

set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r02x_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r02x_pytest_gpu.log; grep -v ": ok" gpurun_out/checked_run.log | tail -3
for c in c3 c4; do timeout 900 ncu --set full --clock-control none -k regex:"fft_|finish_kernel" -c 5 -o gpurun_out/r02x_aux_$c python tools/prof_apply.py $c 1 > gpurun_out/r02x_aux_$c.log 2>&1; echo ncu_$c=$?; done
for D in 2048 4096; do for cl in 0 1; do echo "CL=$cl"; REXI_FFT_CL=$cl python tools/time_fft.py $D; done; done
for c in c3 c4; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_r02x.json 2> gpurun_out/bench_${c}_r02x.err; done

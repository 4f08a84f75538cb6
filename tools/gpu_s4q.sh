# persistent prefetching cluster column passes (fft_cols_clp_kernel) vs fft_cols_cl_kernel
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fft or 4096 or 2048 or c4" > gpurun_out/s4q_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/s4q_pytest.log
timeout 300 python tools/race_probe.py 4096 3; timeout 300 python tools/race_probe.py 2048 3
for v in 0 1 0 1; do for D in 2048 4096; do REXI_FFT_CLP=$v python tools/time_fft_apply.py $D | sed "s/^/clp=$v /"; done; done
timeout 900 python -m pytest tests/test_gpu_checked.py -q > gpurun_out/s4q_checked.log 2>&1; echo checked_rc=$?; tail -1 gpurun_out/checked_run.log
timeout 900 ncu --set full --clock-control none -k regex:"fft_cols_cl" -c 2 -o gpurun_out/s4q_clp python tools/prof_apply.py c4 1 > gpurun_out/s4q_ncu.log 2>&1; echo ncu=$?

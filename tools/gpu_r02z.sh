set -x
for i in 2 1; do REXI_FFT_CLI=$i python -m pytest tests/test_gpu_parity.py -q -x -k "fft_4096 or fft_sampled" 2>&1 | tail -1; REXI_FFT_CLI=$i python tools/race_probe.py 4096 2; done
for D in 2048 4096; do for i in 1 2; do echo "CLI=$i"; REXI_FFT_CLI=$i python tools/time_fft.py $D; done; done
for i in 1 2; do REXI_FFT_CLI=$i timeout 900 ncu --set full --clock-control none -k regex:"fft_cols" -c 2 -o gpurun_out/r02z_cols_c4_i$i python tools/prof_apply.py c4 1 > gpurun_out/r02z_cols_c4_i$i.log 2>&1; done

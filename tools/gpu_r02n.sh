mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fft or apply_vs_oracle or full_size" > gpurun_out/pytest_fft_r02n.log 2>&1; echo pytest_fft_rc=$?
tail -3 gpurun_out/pytest_fft_r02n.log
for D in 512 1024 2048 4096 8192; do
  for cfg in "REXI_FFT_R16=0 REXI_FFT_C16=0" "REXI_FFT_R16=1 REXI_FFT_C16=0" "REXI_FFT_R16=0 REXI_FFT_C16=1" "REXI_FFT_R16=1 REXI_FFT_C16=1"; do
    echo "$cfg"; env $cfg timeout 120 python tools/time_fft.py $D
  done
done 2>&1 | tee gpurun_out/fft16_r02n.log

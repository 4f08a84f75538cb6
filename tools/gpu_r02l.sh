mkdir -p gpurun_out
for D in 512 1024 2048 4096; do
  for R in 1 2 4 8; do echo "ROWS=$R"; REXI_FFT_ROWS=$R timeout 120 python tools/time_fft.py $D; done
  for C in 1 2 4 8; do echo "COLS=$C"; REXI_FFT_COLS=$C timeout 120 python tools/time_fft.py $D; done
done 2>&1 | tee gpurun_out/fft_tune_r02l.log

set -x
for c in c3 c4; do timeout 900 ncu --set full --clock-control none -k regex:"fft_cols" -c 2 -o gpurun_out/r02w_aux_$c python tools/prof_apply.py $c 1 > gpurun_out/r02w_aux_$c.log 2>&1; echo ncu_$c=$?; done
for D in 1024 2048 4096; do for cl in 0 1; do echo "CL=$cl"; REXI_FFT_CL=$cl python tools/time_fft.py $D; done; done

set -x
mkdir -p gpurun_out
for D in 1024 4096; do
timeout 900 ncu --set full --clock-control none -k regex:fft_ -c 4 -o gpurun_out/r02j_fft_$D python tools/prof_fft.py $D > gpurun_out/r02j_fft_$D.log 2>&1; echo ncu_$D=$?
python tools/time_fft.py $D
done
python tools/time_fft.py 512
python tools/time_fft.py 2048

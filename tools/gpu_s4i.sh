# C4: ten-step run to T = 10, launch list, and a full capture of the bulk-staged pole kernel
set -x
mkdir -p gpurun_out
python examples/lrsw_gaussian.py 4096 1.0 10 > gpurun_out/s4i_c4_multistep10.txt 2>&1; echo ex_rc=$?
cat gpurun_out/s4i_c4_multistep10.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4i_c4_launches.csv python tools/prof_apply.py c4 1 > gpurun_out/s4i_ncu1.log 2>&1; echo ncu1=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pole_kernel -c 1 -o gpurun_out/s4i_c4_pole python tools/prof_apply.py c4 1 > gpurun_out/s4i_ncu2.log 2>&1; echo ncu2=$?

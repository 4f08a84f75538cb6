set -x
mkdir -p gpurun_out
python tools/time_partial.py c2 200 > gpurun_out/s4c_partial_c2.jsonl 2>&1; echo rc=$?
python tools/time_partial.py c3 100 > gpurun_out/s4c_partial_c3.jsonl 2>&1; echo rc=$?
python tools/time_partial.py c4 3 > gpurun_out/s4c_partial_c4.jsonl 2>&1; echo rc=$?
cat gpurun_out/s4c_partial_c*.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4c_c2_partial_launches.csv python tools/time_partial.py c2 3 > gpurun_out/s4c_ncu.log 2>&1; echo ncu=$?

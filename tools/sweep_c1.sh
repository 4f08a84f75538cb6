# C1 fused-step timing (tools/time_step_events.py) and stage marks
python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -2
python tools/time_step_events.py c1 400 2>&1 | grep "timing=0 flush=[12]"
python tools/time_step_events.py c1 400 2>&1 | grep "timing=0 flush=[12]"
REXI_SMALL_TRACE=1 python tools/trace_c1.py 2> gpurun_out/trace_c1.log; tail -4 gpurun_out/trace_c1.log

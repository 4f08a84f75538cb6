# C1 fused-step timing sweep (tools/time_step_events.py)
python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -2
REXI_SMALL_NC=3 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -2
for v in "REXI_SMALL_NC=1" "REXI_SMALL_NC=2" "REXI_SMALL_NC=3" "REXI_SMALL_NC=4" "REXI_SMALL_NC=6"; do
  echo "== $v"; env $v python tools/time_step_events.py c1 400 2>&1 | grep "timing=0 flush=[12]"
done
REXI_SMALL_NC=4 REXI_SMALL_TRACE=1 python tools/trace_c1.py 2> gpurun_out/trace_c1_nc4.log; tail -4 gpurun_out/trace_c1_nc4.log
REXI_SMALL_NC=1 REXI_SMALL_TRACE=1 python tools/trace_c1.py 2> gpurun_out/trace_c1_nc1.log; tail -4 gpurun_out/trace_c1_nc1.log

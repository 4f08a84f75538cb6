# C1 fused-step timing sweep (tools/time_step_events.py)
python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -2
REXI_SMALL_NC=4 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -2
for v in "REXI_SMALL_NC=1" "REXI_SMALL_NC=2" "REXI_SMALL_NC=3" "REXI_SMALL_NC=4"; do
  echo "== $v"; env $v python tools/time_step_events.py c1 400 2>&1 | grep "timing=0 flush=[12]"
done
for nc in ${SWEEP_NCS:-1}; do
for st in -2 -1 0 1 2 3 4 99; do echo "== NC $nc stop $st"; REXI_SMALL_NC=$nc REXI_SMALL_STOP=$st python tools/time_step_events.py c1 400 2>&1 | grep "timing=0 flush=[12]"; done
done

for k in -2 -1 0 1; do echo "STOP=$k"; REXI_SMALL_STOP=$k timeout 120 python tools/time_c1.py 64 0.02; done 2>&1 | tee gpurun_out/c1_stages_r02s.log

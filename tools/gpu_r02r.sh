for k in 0 1 2 3 4 5 99; do echo "STOP=$k"; REXI_SMALL_STOP=$k timeout 120 python tools/time_c1.py 64 0.02; done 2>&1 | tee gpurun_out/c1_stages_r02r.log

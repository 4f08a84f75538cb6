timeout 600 python tools/tune.py c2 pfhx > gpurun_out/tune_c2_r02t.jsonl 2>&1; cat gpurun_out/tune_c2_r02t.jsonl

set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r02m.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_r02m.log
timeout 900 python tests/scripts/sweep.py 512 > gpurun_out/r02_sweep_c5_512.jsonl 2> gpurun_out/sweep.err; echo sweep_rc=$?
timeout 600 python tests/scripts/paper_rows.py > gpurun_out/r02_paper_rows.jsonl 2> gpurun_out/rows.err; echo rows_rc=$?
timeout 600 python examples/lrsw_gaussian.py 4096 1.0 5 > gpurun_out/r02_c4_multistep.txt 2>&1; echo ex_rc=$?
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_r02m.json 2> gpurun_out/bench_c4_r02m.err
timeout 600 python bench.py --steps 100 --warmup 10 > gpurun_out/bench_c2_r02m.json 2> gpurun_out/bench_c2_r02m.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ref_c2_r02m.json 2> gpurun_out/ref_c2_r02m.err
cat gpurun_out/ref_c2_r02m.json | cut -c1-300

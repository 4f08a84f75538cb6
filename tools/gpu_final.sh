# Final validation of the round (run under gpurun): GPU suite, smoke, bench lines C1..C4,
# ncu launch list + pole-kernel capture of the C2 bench, fused C1 capture, FFT passes at 4096^2.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fin_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/fin_pytest_gpu.log; tail -1 gpurun_out/checked_run.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo smoke_rc=$?
python bench.py > gpurun_out/fin_bench_c2.json 2> gpurun_out/fin_bench_c2.err; echo c2_rc=$?
python bench.py --config c1 > gpurun_out/fin_bench_c1.json 2> gpurun_out/fin_bench_c1.err; echo c1_rc=$?
python bench.py --config c3 --no-cpu-baseline > gpurun_out/fin_bench_c3.json 2> gpurun_out/fin_bench_c3.err; echo c3_rc=$?
python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/fin_bench_c4.json 2> gpurun_out/fin_bench_c4.err; echo c4_rc=$?
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/fin_ref_c2.json 2> gpurun_out/fin_ref_c2.err; echo ref_rc=$?
bash tools/gpu_profile.sh fin_c2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_small2 -s 5 -c 1 -o gpurun_out/fin_c1_small python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fin_ncu_c1.log 2>&1; echo ncu_c1=$?
timeout 900 ncu --set full --clock-control none -k regex:"fft_|finish_kernel" -c 5 -o gpurun_out/fin_aux_c4 python tools/prof_apply.py c4 1 > gpurun_out/fin_aux_c4.log 2>&1; echo ncu_c4=$?

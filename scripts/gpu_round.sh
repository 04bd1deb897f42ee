# Full round evidence: GPU tests, smoke, bench lines, ncu launch list + full capture.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo PYTEST $?
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE $?
timeout -s KILL 400 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo BENCH_C2 $?
timeout -s KILL 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo BENCH_C1 $?
timeout -s KILL 600 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo BENCH_C3 $?
timeout -s KILL 600 python bench.py --config c3bf16 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3bf16.json 2> gpurun_out/bench_c3bf16.err; echo BENCH_C3BF16 $?
timeout -s KILL 300 python bench.py --impl reference --steps 10 --warmup 2 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo BENCH_REF $?
timeout -s KILL 200 python scripts/prof_layer.py --config c2 --iters 8 > gpurun_out/plain_launch.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python scripts/prof_layer.py --config c2 --iters 8 > gpurun_out/ncu_launch.log 2>&1; echo NCU_LAUNCH $?
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:kan_gather -s 2 -c 1 -o gpurun_out/prof_c2_l0 python scripts/prof_layer.py --config c2 --iters 4 > gpurun_out/ncu_c2.log 2>&1; echo NCU_C2 $?
timeout -s KILL 200 python scripts/prof_layer.py --config c3 --iters 2 > gpurun_out/plain_c3.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:kan_gather -s 1 -c 1 -o gpurun_out/prof_c3_l0 python scripts/prof_layer.py --config c3 --iters 2 > gpurun_out/ncu_c3.log 2>&1; echo NCU_C3 $?
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log

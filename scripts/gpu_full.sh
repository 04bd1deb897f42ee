cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/t2.log 2>&1; echo PYTEST $?
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE $?
timeout -s KILL 300 python bench.py --steps 20000 --warmup 200 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo BENCH_C2 $?
timeout -s KILL 300 python bench.py --config c1 --steps 20000 --warmup 200 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo BENCH_C1 $?
timeout -s KILL 400 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo BENCH_C3 $?
timeout -s KILL 400 python bench.py --config c3bf16 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3bf16.json 2> gpurun_out/bench_c3bf16.err; echo BENCH_C3BF16 $?
timeout -s KILL 300 python bench.py --steps 64 --warmup 16 --no-cpu-baseline > gpurun_out/plain_c2.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 64 --warmup 16 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo NCU1 $?
tail -3 gpurun_out/t2.log; cat gpurun_out/smoke.log | tail -3
for f in gpurun_out/bench_*.json; do echo $f; cat $f | head -c 3000; echo; done
tail -5 gpurun_out/bench_c2.err

# one GPU round trip: GPU tests, then the listed bench configs (args: configs)
set -x
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
for c in "$@"; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
  tail -3 gpurun_out/bench_$c.err
done

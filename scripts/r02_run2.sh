set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config c5pc --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c5pc.json 2> gpurun_out/bench_c5pc.err; echo "c5pc rc=$?"
timeout 900 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
timeout 900 python bench.py --impl reference --config c5 --steps 3 --warmup 1 > gpurun_out/bench_ref_c5.json 2> gpurun_out/bench_ref_c5.err; echo "ref rc=$?"
tail -3 gpurun_out/*.err

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02_pytest_gpu.log
timeout 600 python bench.py --config c5 --steps 20 --warmup 5 > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err; echo "c5 rc=$?"
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err; echo "c2 rc=$?"
cat gpurun_out/r02_bench_c5.json | head -c 3000

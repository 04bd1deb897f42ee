set -x
python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/val_bench_c5.json 2> gpurun_out/val_bench_c5.err; echo "bench rc=$?"
cat gpurun_out/val_bench_c5.json
timeout 2700 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log

set -x
python scripts/prof_layer.py --config c5 --batch 2048 --iters 3 --opt convw_tr=2 2>&1 | sed -n '2,5p;8,10p'
timeout 900 python bench.py --config c5 --steps 20 --warmup 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
tail -2 gpurun_out/bench_c5.err
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log

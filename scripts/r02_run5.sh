set -x
python scripts/prof_layer.py --config c5 --batch 2048 --iters 5 2>&1 | tee gpurun_out/prof_c5.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log

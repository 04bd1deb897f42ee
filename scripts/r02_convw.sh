set -x
timeout 900 python -m pytest tests/test_gpu_conv.py -q -x -p no:cacheprovider -k "convw" > gpurun_out/pytest_convw.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/pytest_convw.log
python scripts/prof_layer.py --config c5 --batch 2048 --iters 5 2>&1 | tee gpurun_out/prof_c5.log

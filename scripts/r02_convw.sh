set -x
timeout 900 python -m pytest tests/test_gpu_conv.py -q -x -p no:cacheprovider -k "convw" > gpurun_out/pytest_convw.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/pytest_convw.log
python scripts/prof_layer.py --config c5 --batch 2048 --iters 5 2>&1 | tee gpurun_out/prof_c5.log
for o in convw_bn=256 convw_mc=2; do echo "opt $o"; python scripts/prof_layer.py --config c5 --batch 2048 --iters 3 --opt $o 2>&1 | sed -n '2,5p;8,10p;13,15p;18,20p'; done

set -x
timeout 1200 python -m pytest tests/test_gpu_conv.py -m gpu -q -x -p no:cacheprovider -k "convw or conv3" > gpurun_out/pytest_convw.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_convw.log
timeout 600 python bench.py --config c4 --steps 200 --warmup 10 > gpurun_out/c4.json 2> gpurun_out/c4.err; echo "c4 rc=$?"
cat gpurun_out/c4.json | cut -c1-1500
timeout 600 python bench.py --config c4 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --opt no_convw=1 > gpurun_out/c4_noconvw.json 2>> gpurun_out/c4.err; echo "c4b rc=$?"
cat gpurun_out/c4_noconvw.json | cut -c1-400
timeout 900 python bench.py --config c5pc --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c5pc.json 2> gpurun_out/c5pc.err; echo "c5pc rc=$?"
cat gpurun_out/c5pc.json | cut -c1-3000

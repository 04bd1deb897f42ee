set -x
for o in "convw_tr=2" "convw_tr=1" "convw_rings=432" "convw_rings=332" "convw_rings=423" "convw_rings=323" "convw_rings=233"; do
  echo "== $o"
  timeout 300 python bench.py --config c4 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --opt $o 2>>gpurun_out/c4tune.err | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['per_launch']['avg_ms'], d['timing']['launch_plan'][-1])"
done
timeout 900 python -m pytest tests/test_gpu_bench_configs.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_bc.log 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/pytest_bc.log

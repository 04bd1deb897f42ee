set -x
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r02_bench_c5.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['whole_forward']['frac'], d['e2e']['value'], d['clocks'])
print([round(x,2) for x in d['roofline']['layer_avg_ms']])"

timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_configs.py -m gpu -q -p no:cacheprovider 2>&1 | tail -12
for c in c2 c1; do
timeout 300 python bench.py --config $c --steps 240 --warmup 24 --no-cpu-baseline --no-e2e 2>>gpurun_out/fuse.err | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], d['value'], d['ms_per_step'], d['roofline']['frac'], d['timing'].get('single_batch_ms'), d['timing']['launch_plan'])"
done
for s in 1 4; do echo "== prof c2 split $s"; python scripts/prof_layer.py --config c2 --split $s --iters 20; done
python scripts/timeline.py --config c2 --split 1 | tail -12

timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "fused" 2>&1 | tail -5
for o in "fuse_persistent=0" "fuse_persistent=1"; do
for s in 1 0; do echo "== prof c2 split $s $o"; python scripts/prof_layer.py --config c2 --split $s --iters 20 --opt $o | tr '\n' ' '; echo; done
for c in c2 c1; do
timeout 300 python bench.py --config $c --steps 240 --warmup 24 --no-cpu-baseline --no-e2e --opt $o 2>>gpurun_out/fuse.err | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], d['value'], d['ms_per_step'], d['roofline']['frac'], d['timing'].get('single_batch_ms'), d['timing']['launch_plan'])"
done
done

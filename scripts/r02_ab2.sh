# A/B of a compile-time variant (args: extra nvcc flags): parity tests of variant B + per-layer times of both
set -x
python scripts/prof_layer.py --config c5 --batch 2048 --iters 5 > gpurun_out/ab_a.log 2>&1
KAN_EXTRA_NVFLAGS="$*" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_conv.py -q -x -p no:cacheprovider -k "convw" 2>&1 | tail -2
python scripts/prof_layer.py --config c5 --batch 2048 --iters 5 > gpurun_out/ab_b.log 2>&1
paste gpurun_out/ab_a.log gpurun_out/ab_b.log

# A/B of a compile-time variant on the C5 layer times: args = extra nvcc flags of variant B
set -x
python scripts/prof_layer.py --config c5 --batch 2048 --iters 3 > gpurun_out/ab_a.log 2>&1
KAN_EXTRA_NVFLAGS="$*" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
python scripts/prof_layer.py --config c5 --batch 2048 --iters 3 > gpurun_out/ab_b.log 2>&1
paste gpurun_out/ab_a.log gpurun_out/ab_b.log

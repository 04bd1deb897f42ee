cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/epi
for s in 0 1; do KAN_EPI_STAGE=$s timeout -s KILL 300 python scripts/prof_layer.py --config c5 --iters 3 > gpurun_out/epi/c5_layers_stg$s.txt 2>&1; done
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q > gpurun_out/epi/pytest.txt 2>&1
tail -3 gpurun_out/epi/pytest.txt
timeout -s KILL 300 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/epi/c5_bench.json 2>gpurun_out/epi/c5_bench.err
cut -c1-250 gpurun_out/epi/c5_bench.json

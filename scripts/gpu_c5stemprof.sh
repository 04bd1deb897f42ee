cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof3
timeout -s KILL 200 python scripts/prof_layer.py --config c5 --iters 1 --nograph --batch 1024 > /dev/null 2>&1 && timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:kan_gather -s 0 -c 1 -o gpurun_out/prof3/c5_stem python scripts/prof_layer.py --config c5 --iters 1 --nograph --batch 1024 > gpurun_out/prof3/ncu.log 2>&1; echo "CAP $?"

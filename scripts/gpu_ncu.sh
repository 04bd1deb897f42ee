cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=${1:-c2}
timeout -s KILL 200 python scripts/prof_layer.py --config $CFG --iters 4 > gpurun_out/plain_$CFG.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:kan_gather -s 2 -c 1 -o gpurun_out/prof_${CFG}_l0 python scripts/prof_layer.py --config $CFG --iters 4 > gpurun_out/ncu_$CFG.log 2>&1; echo NCU $?

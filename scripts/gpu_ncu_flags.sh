cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export KAN_DBG_FLAGS=${2:-0}
CFG=${1:-c2}
timeout -s KILL 200 python scripts/prof_layer.py --config $CFG --iters 4 --split 1 > gpurun_out/plain_f.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:kan_gather -s 2 -c 1 -o gpurun_out/prof_flags python scripts/prof_layer.py --config $CFG --iters 4 --split 1 > gpurun_out/ncu_f.log 2>&1; echo NCU $?

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof2
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof2/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "LAUNCH c2 $?"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof2/launches_c1.csv python bench.py --config c1 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "LAUNCH c1 $?"
timeout -s KILL 200 python scripts/prof_layer.py --config c2 --iters 2 --nograph --split 1 > /dev/null 2>&1 && timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:kan_gather -s 1 -c 1 -o gpurun_out/prof2/c2_l0 python scripts/prof_layer.py --config c2 --iters 2 --nograph --split 1 > /dev/null 2>&1; echo "CAP c2 $?"

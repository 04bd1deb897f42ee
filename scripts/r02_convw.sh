set -x
python scripts/prof_layer.py --config c5 --batch 2048 --iters 3 > gpurun_out/prof_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:convw -s 0 -c 1 -o gpurun_out/prof_convw2 python scripts/prof_layer.py --config c5 --batch 2048 --iters 3 > gpurun_out/ncu_convw.log 2>&1; echo "ncu rc=$?"

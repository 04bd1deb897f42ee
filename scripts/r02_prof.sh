# final C5 bench line + launch list of the bench command + full ncu capture of the dominant kernel
set -x
timeout 900 python bench.py --config c5 --steps 20 --warmup 5 > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --config c5 --steps 3 --warmup 1 > gpurun_out/r02_bench_reference_c5.json 2> gpurun_out/r02_bench_reference_c5.err; echo "ref rc=$?"
python bench.py --config c5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_c5.csv python bench.py --config c5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
python scripts/prof_layer.py --config c5 --iters 1 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:convw -s 3 -c 1 -o gpurun_out/r02_c5_l4 python scripts/prof_layer.py --config c5 --iters 1 > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"

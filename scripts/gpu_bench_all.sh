# One bench line per workload (BASELINE configs 1-5, the fp32 Cox-de Boor
# baseline, the C2 precision sweep, C5 with per-channel weights + SiLU).
#   gpurun --timeout 3000 -- 'bash scripts/gpu_bench_all.sh'
set -x
for c in c1 c1fp32 c2 c2k4 c2k3 c2k2 c2w4 c3 c3bf16 c4 c5pc; do
  steps=200; [ $c = c5pc ] && steps=20
  timeout 900 python bench.py --config $c --steps $steps --warmup 10 --cpu-seconds 5 > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err; echo "$c rc=$?"
  tail -2 gpurun_out/r02_bench_$c.err
done

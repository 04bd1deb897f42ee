# bench lines behind the paper's GPU claims: LUT vs fp32 Cox-de Boor on C1, the C2 precision sweep
set -x
for c in c1 c1fp32 c2 c2k4 c2k3 c2k2 c2w4 c3 c3bf16 c4 c5pc; do
  timeout 900 python bench.py --config $c --steps 200 --warmup 10 --cpu-seconds 5 > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err; echo "$c rc=$?"
  tail -2 gpurun_out/r02_bench_$c.err
done

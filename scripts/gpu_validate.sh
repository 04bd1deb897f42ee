# Round-end validation on one B200: GPU parity suite, smoke, the headline bench
# (C5) and its reference arm, and the bench lines of the two configurations
# that run the SiLU form of kan_convw (C5pc, C4).
#   gpurun --timeout 3600 -- 'bash scripts/gpu_validate.sh'
set -x
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference_c5.json 2> gpurun_out/r02_bench_reference_c5.err; echo "ref rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err; echo "bench rc=$?"
cat gpurun_out/r02_bench_c5.json | head -c 1500
timeout 900 python bench.py --config c5pc --steps 20 --warmup 10 --cpu-seconds 5 > gpurun_out/r02_bench_c5pc.json 2> gpurun_out/r02_bench_c5pc.err; echo "c5pc rc=$?"
timeout 900 python bench.py --config c4 --steps 200 --warmup 10 --cpu-seconds 5 > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; echo "c4 rc=$?"

# spline-table mode: GPU parity tests, bench lines, launch list and one ncu capture
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/st
timeout -s KILL 600 python -m pytest tests/test_gpu_spline_table.py -q --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/st/pytest.log 2>&1; echo "PYTEST $?"; tail -3 gpurun_out/st/pytest.log
for c in c1st c2st c2st4 c4st; do
  timeout -s KILL 300 python bench.py --config $c --steps 3000 --warmup 30 --cpu-seconds 5 > gpurun_out/st/ours_$c.json 2> gpurun_out/st/ours_$c.err; echo "BENCH $c $?"
  python -c "import json;d=json.load(open('gpurun_out/st/ours_$c.json'));r=d['roofline'];print('$c', '%.4g'%d['value'], round(d['ms_per_step']*1e3,2),'us', r['bound'], round(r['frac'],3), [round(v*1e3,2) for v in r['layer_avg_ms']], 'e2e %.3g'%d['e2e']['value'], 'cpu', d['cpu_baseline'] and d['cpu_baseline'].get('value'))" 2>&1 | tail -1
done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/st/launches_c2st.csv python bench.py --config c2st --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "LAUNCH $?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:kan_st_layer -s 4 -c 1 -o gpurun_out/st/c2st_l0 python bench.py --config c2st --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/st/ncu.log 2>&1; echo "CAP $?"

# ncu evidence for profiles/: the launch list of the headline bench command and
# one --set full capture of each config's dominant kernel (each only after the
# same command exited 0 without ncu).   gpurun --timeout 3000 -- 'bash scripts/gpu_profile.sh'
set -x
python bench.py --config c5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_c5.csv python bench.py --config c5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
cap() {  # name config kernel-regex skip [extra prof_layer args]
  local name=$1 cfg=$2 rx=$3 skip=$4; shift 4
  python scripts/prof_layer.py --config $cfg --iters 1 "$@" > gpurun_out/plain_$name.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -f -o gpurun_out/$name python scripts/prof_layer.py --config $cfg --iters 1 "$@" > gpurun_out/ncu_$name.log 2>&1; echo "$name rc=$?"
}
cap r02_c5_l2 c5 convw 1          # stage-1 conv, residual add, fp32 + levels sidecar out (the bench's dominant launch)
cap r02_c5_l4 c5 convw 3          # stage-1 conv, residual add, levels out
cap r02_c5_l8 c5 convw 7          # stage-2 conv, levels out (N = 128)
cap r02_c5_l13 c5 convw 9         # stage-3 conv, levels out (two N tiles: two MMA-issuing warps)
cap r02_c4_conv c4 convw 0        # C4: SiLU form, NCHW output
cap r02_c3_l0 c3 gather 0         # C3 int8 layer 0
cap r02_c3bf16_l0 c3bf16 gather 0 # C3 bf16 layer 0
cap r02_c2_l0 c2 gather 0 --split 1   # C2 bench configuration (unsplit)
# DRAM bytes of EVERY kan_convw launch of one C5 forward (one light pass): the
# per-launch average behind roofline.traffic of the kernel-level roofline
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:convw -c 14 --csv --log-file gpurun_out/r02_c5_convw_dram.csv python scripts/prof_layer.py --config c5 --iters 1 > gpurun_out/ncu_convw_dram.log 2>&1; echo "convw dram rc=$?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gather -c 3 --csv --log-file gpurun_out/r02_c3_gather_dram.csv python scripts/prof_layer.py --config c3 --iters 1 > gpurun_out/ncu_c3_dram.log 2>&1; echo "c3 dram rc=$?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gather -c 3 --csv --log-file gpurun_out/r02_c3bf16_gather_dram.csv python scripts/prof_layer.py --config c3bf16 --iters 1 > gpurun_out/ncu_c3bf16_dram.log 2>&1; echo "c3bf16 dram rc=$?"
# summarise on the box (the .ncu-rep files are too large to travel): details
# pages + ncu_summary.json via make_profiles.py, stall/instruction summaries
python scripts/make_profiles.py gpurun_out c5_l2=r02_c5_l2 c5_l4=r02_c5_l4 c5_l8=r02_c5_l8 c5_l13=r02_c5_l13 c4_l0=r02_c4_conv c3_l0=r02_c3_l0 c3bf16_l0=r02_c3bf16_l0 c2_l0=r02_c2_l0
for n in r02_c5_l2 r02_c5_l4 r02_c5_l8 r02_c5_l13 r02_c4_conv r02_c3_l0 r02_c3bf16_l0 r02_c2_l0; do
  cp profiles/$n.txt gpurun_out/
  python scripts/ncu_summary.py gpurun_out/$n.ncu-rep --tensor > gpurun_out/${n}_stalls.txt 2>&1
  ncu -i gpurun_out/$n.ncu-rep --page raw --csv > gpurun_out/${n}_raw.csv 2>/dev/null
  rm -f gpurun_out/$n.ncu-rep
done
python scripts/make_profiles.py --dram-csv c5_convw=gpurun_out/r02_c5_convw_dram.csv c3_gather=gpurun_out/r02_c3_gather_dram.csv c3bf16_gather_bf16=gpurun_out/r02_c3bf16_gather_dram.csv
cp profiles/ncu_summary.json gpurun_out/

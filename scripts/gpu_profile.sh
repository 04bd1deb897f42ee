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
cap r02_c5_l4 c5 convw 3          # stage-1 conv with residual + fp32/sidecar output (the bench's dominant launch)
cap r02_c5_l8 c5 convw 7          # stage-2 conv, levels out (N = 128)
cap r02_c4_conv c4 convw 0        # C4: SiLU form, NCHW output
cap r02_c3_l0 c3 gather 0         # C3 int8 layer 0
cap r02_c3bf16_l0 c3bf16 gather 0 # C3 bf16 layer 0
cap r02_c2_l0 c2 gather 0 --split 1   # C2 bench configuration (unsplit)

cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_conv.py -q -p no:cacheprovider -k "bf16" 2>&1 | tail -2
timeout -s KILL 300 python scripts/prof_layer.py --config c3bf16 --iters 3 2>&1 | tail -4 | head -3

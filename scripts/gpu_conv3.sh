cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python -m pytest tests/test_gpu_conv.py -q -x --timeout 60 --timeout-method=thread -p no:cacheprovider -k "conv3" > /tmp/t3.log 2>&1; echo PYTEST3 $?; grep -E "passed|failed|Error|^E " /tmp/t3.log | head -8

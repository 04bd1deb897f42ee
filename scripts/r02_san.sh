# compute-sanitizer on small forwards of every kernel family (one tool per call: $1)
set -x
python scripts/sanitize_small.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?"
tail -2 gpurun_out/san_plain.log
timeout 1500 compute-sanitizer --tool $1 --print-limit 20 python scripts/sanitize_small.py > gpurun_out/san_$1.log 2>&1; echo "$1 rc=$?"
tail -15 gpurun_out/san_$1.log

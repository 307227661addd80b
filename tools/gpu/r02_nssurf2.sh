# (experiment, not kept) with the momentum register cap: Kuhn surface rows on a third stream x boundary CTA size: 2.791-2.806 vs 2.785 ms
for rep in 1 2; do
for v in "0 128" "1 128" "1 64" "1 32"; do
  set -- $v
  echo "== surf $1 bthreads $2"
  FPB_NS_SURF=$1 FPB_TUNE_KGRAD_BTHREADS=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'], d['kernels_ms'])"
done
done
FPB_NS_SURF=1 FPB_TUNE_KGRAD_BTHREADS=32 timeout 600 python -m pytest tests/test_gpu_kuhn.py -q -m gpu -k "ns_d" -p no:cacheprovider 2>&1 | tail -1

# (experiment, reverted) assemble_ns_d with the Kuhn surface rows on a third stream: FPB_NS_SURF 0/1/2 x boundary CTA size; no gain (2.841-2.934 vs 2.846 ms)
for v in "0 128" "1 128" "1 64" "2 64" "2 32" "1 32"; do
  set -- $v
  echo "== surf $1 bthreads $2"
  FPB_NS_SURF=$1 FPB_TUNE_KGRAD_BTHREADS=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'], d['kernels_ms'])"
done
FPB_NS_SURF=2 timeout 600 python -m pytest tests/test_gpu_kuhn.py -q -m gpu -k "ns_d" -p no:cacheprovider 2>&1 | tail -1

# (experiment, not kept) Kuhn B_xyz surface rows before the interior lines in the two-stream NS step: 2.848-2.851 vs 2.804-2.806 ms (lines first kept);
# the per-stream finish times vary run to run (the CTA scheduler interleaves the two streams differently)
timeout 900 python -m pytest tests/test_gpu_kuhn.py tests/test_distributed_solver.py -q -m gpu -p no:cacheprovider 2>&1 | tail -1
for v in 1 0 1 0; do
  echo "== surface first $v"
  FPB_KUHN_SURFACE_FIRST=$v timeout 600 python tools/ns_timeline.py 2>&1 | head -1
  FPB_KUHN_SURFACE_FIRST=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'], d['kernels_ms'])"
done

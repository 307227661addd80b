# compute-sanitizer on the Kuhn-box kernels (momentum / scalar3 pencils, B_xyz lines + boundary rows, slab ranges)
mkdir -p gpurun_out
K='oracle or wide or scalar3_matches_oracle or gradients'
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python -m pytest tests/test_gpu_kuhn.py -q -m gpu -p no:cacheprovider -k "$K" > gpurun_out/kuhn_memcheck.log 2>&1; echo memcheck_rc=$?; grep -E "ERROR SUMMARY|passed|failed|Invalid" gpurun_out/kuhn_memcheck.log | head -8
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_kuhn.py -q -m gpu -p no:cacheprovider -k "$K" > gpurun_out/kuhn_racecheck.log 2>&1; echo racecheck_rc=$?; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|hazard" gpurun_out/kuhn_racecheck.log | head -10
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_kuhn.py -q -m gpu -p no:cacheprovider -k "$K" > gpurun_out/kuhn_synccheck.log 2>&1; echo synccheck_rc=$?; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/kuhn_synccheck.log | head -5
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests/test_gpu_kuhn.py -q -m gpu -p no:cacheprovider -k "oracle and not jitter" > gpurun_out/kuhn_initcheck.log 2>&1; echo initcheck_rc=$?; grep -E "ERROR SUMMARY|passed|failed|Uninitialized" gpurun_out/kuhn_initcheck.log | head -5

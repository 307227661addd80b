# round 2: the reference suite through the package, then the full gpu suite
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_reference_suite.py -q -m gpu -p no:cacheprovider -s > gpurun_out/pytest_refsuite.log 2>&1; tail -3 gpurun_out/pytest_refsuite.log
grep -E "passed|failed" gpurun_out/refsuite.log | tail -2
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider --deselect tests/test_reference_suite.py > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log

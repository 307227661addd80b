# round 2: reference suite through the package + parity at config sizes
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 1500 python -m pytest tests/test_reference_suite.py -q -m gpu -p no:cacheprovider -s > gpurun_out/pytest_refsuite.log 2>&1; tail -3 gpurun_out/pytest_refsuite.log
grep -E "passed|failed" gpurun_out/refsuite.log | tail -2
timeout 2400 python -m pytest tests/test_gpu_scale.py -q -m gpu -p no:cacheprovider --durations=0 > gpurun_out/pytest_scale.log 2>&1; tail -15 gpurun_out/pytest_scale.log

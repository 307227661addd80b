mkdir -p gpurun_out
for m in p2p; do NCCL_DEBUG=INFO NCCL_DEBUG_FILE=gpurun_out/nccl_$m.log timeout 60 python tools/native_probe.py $m > gpurun_out/native_probe_$m.log 2>&1; echo $m rc=$?; tail -4 gpurun_out/native_probe_$m.log; done
timeout 300 python -m pytest tests/test_native_halo.py -q -m gpu -p no:cacheprovider 2>&1 | tail -3

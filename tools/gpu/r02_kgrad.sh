mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kuhn.py -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_kuhn.log 2>&1; tail -3 gpurun_out/pytest_kuhn.log
for t in kgrad_kchunk=0; do
  echo "== $t"; timeout 600 python tools/kmom_probe.py --kchunks 0 --blocks 0 --grad 1 --tune $t 2>&1 | grep grad_
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_kuhn_grad" -s 4 -c 2 -o gpurun_out/prof_kgrad python tools/kmom_probe.py --sizes 256x256x256 --reps 1 --blocks 0 --grad 1 > gpurun_out/ncu_kgrad.log 2>&1; tail -1 gpurun_out/ncu_kgrad.log

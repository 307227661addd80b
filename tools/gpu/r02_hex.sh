mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_distorted.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_distorted.log 2>&1; tail -3 gpurun_out/pytest_distorted.log
for R in 64 32; do timeout 600 python tools/hexprobe.py --canon-rows $R > gpurun_out/hexprobe_$R.json 2> gpurun_out/hexprobe.err; cat gpurun_out/hexprobe_$R.json; tail -3 gpurun_out/hexprobe.err; done
FPB_HEX_MORTON=0 timeout 600 python tools/hexprobe.py --canon-rows 32 > gpurun_out/hexprobe_nat.json 2>&1; cat gpurun_out/hexprobe_nat.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hex_rows_canon -s 1 -c 1 -o gpurun_out/prof_hex python tools/hexprobe.py --reps 1 --canon-rows 64 > gpurun_out/ncu_hex.log 2>&1; tail -2 gpurun_out/ncu_hex.log

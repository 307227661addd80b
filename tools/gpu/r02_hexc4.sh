# HEX08 box: parity tests + C4 block of the bench
timeout 900 python -m pytest tests -q -m gpu -k "hex" -p no:cacheprovider 2>&1 | tail -1
timeout 900 python tools/hexprobe.py --reps 7 2>&1 | tail -1 | grep -o '"once_ms.*'
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-solver > gpurun_out/bench_c4.json 2>gpurun_out/bench_c4.err; python -c "
import json;d=json.load(open('gpurun_out/bench_c4.json'));c=d['configs']['c4'];print(d['ms_per_step'], c.get('ms_per_step'), c.get('kernels_ms'))"

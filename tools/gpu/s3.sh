timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 900 python bench.py --no-cpu-baseline --no-solver > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step']); c=d['configs']; print(json.dumps(c['c3'])[:600]); print(c['c4']['ms_per_step'], json.dumps(c['c4']['kernels'])[:700])"

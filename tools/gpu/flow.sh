timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 600 python tools/flow_probe.py 2>&1 | tail -1
timeout 600 python tools/flow_probe.py --max-padding 0 2>&1 | tail -1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value']); print(json.dumps(d['configs']['flow'])[:900]); print({k: (round(v['ms'],4), round(v.get('frac_hbm', 0),3), v.get('ms_per_iter')) for k,v in d['solver'].items()})"

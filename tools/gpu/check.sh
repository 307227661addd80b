timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 1500 gpurun_out/bench.json

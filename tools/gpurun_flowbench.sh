mkdir -p gpurun_out
timeout 600 python -c "
import sys, json; sys.path.insert(0, '.')
import bench
print(json.dumps(bench.flow_block(94, 94, 95), indent=1))
" 2>&1 | tail -30

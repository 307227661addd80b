"""Step-by-step probe of the compiled NCCL halo on one GPU (development aid)."""
import datetime
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def log(*a):
    print(f"[{time.time():.1f}]", *a, flush=True)


torch.cuda.set_device(0)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0),
                        timeout=datetime.timedelta(seconds=60))
log("pg up")
from paper_2107_11541_b200.distributed import NativeComm  # noqa: E402

nc = NativeComm()
log("comm up", nc.ptr)
x = torch.arange(200, dtype=torch.float64, device="cuda")
r = torch.tensor([1.5, -2.0], dtype=torch.float64, device="cuda")
nc.allreduce(r)
torch.cuda.synchronize()
log("allreduce", r.tolist())
nc.exchange([(0, 0, 120, 10)], x, False)
torch.cuda.synchronize()
log("copy", x[120:123].tolist())
nc.exchange([(0, 0, 0, 10)], x, True)
torch.cuda.synchronize()
log("sum", x[:3].tolist())
y = torch.ones(64, dtype=torch.float64, device="cuda")
g = torch.cuda.CUDAGraph()
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
mode = sys.argv[1] if len(sys.argv) > 1 else "both"
log("capture", mode)
with torch.cuda.graph(g, stream=side):
    if mode in ("both", "p2p"):
        nc.exchange([(0, 0, 0, 16)], y, True)
    if mode in ("both", "ar"):
        nc.allreduce(y[32:40])
torch.cuda.current_stream().wait_stream(side)
log("captured")
g.replay()
torch.cuda.synchronize()
log("replayed", y[:2].tolist())
del g
torch.cuda.synchronize()
log("graph freed")
nc.close()
log("comm closed")
dist.destroy_process_group()
log("done")

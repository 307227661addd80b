"""The compiled NCCL halo path (halo.cu: fpb_nccl_comm_init,
fpb_halo_exchange, fpb_allreduce_sum — SURVEY.md 8(b) `fpb_halo_sum`),
driven through distributed.NativeComm on the box's one GPU: a one-rank NCCL
group whose segments name rank 0 itself (NCCL send/recv to self), so the
group/send/recv/add path runs for real; then the same exchange captured in
a CUDA graph and replayed.  Multi-rank correctness of the segment order is
the same code as the gloo tests' (tests/test_distributed*.py)."""

import datetime
import os
import tempfile
import traceback

import pytest
import torch

pytestmark = pytest.mark.gpu


def _worker(initfile, q):
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"file://{initfile}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0), timeout=datetime.timedelta(seconds=120))
    try:
        from paper_2107_11541_b200.distributed import NativeComm, native_comm

        nc = native_comm()
        assert isinstance(nc, NativeComm)
        x = torch.arange(200, dtype=torch.float64, device="cuda")
        want = x.clone()
        want[0:10] *= 2.0
        want[50:57] *= 2.0
        nc.exchange([(0, 0, 0, 10), (0, 50, 50, 7)], x, True)  # sum: mine + "peer's" (= mine)
        torch.cuda.synchronize()
        ok_sum = bool(torch.equal(x, want))
        nc.exchange([(0, 0, 120, 10)], x, False)  # copy into a ghost range
        want[120:130] = want[0:10]
        torch.cuda.synchronize()
        ok_copy = bool(torch.equal(x, want))
        r = torch.tensor([1.5, -2.0], dtype=torch.float64, device="cuda")
        nc.allreduce(r)
        ok_red = r.tolist() == [1.5, -2.0]
        # captured once, replayed twice
        y = torch.ones(64, dtype=torch.float64, device="cuda")
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=side):
            nc.exchange([(0, 0, 0, 16)], y, True)
            nc.allreduce(y[32:40])
        torch.cuda.current_stream().wait_stream(side)
        g.replay()
        g.replay()
        torch.cuda.synchronize()
        ok_graph = bool((y[:16] == 4.0).all() and (y[16:] == 1.0).all())
        del g  # a graph holding captured NCCL work must go before its communicator
        torch.cuda.synchronize()
        nc.close()
        q.put({"sum": ok_sum, "copy": ok_copy, "allreduce": ok_red, "graph": ok_graph})
    except Exception:
        q.put(traceback.format_exc())
    finally:
        dist.destroy_process_group()


def test_native_nccl_halo_one_rank(cuda_ok):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as d:
        p = ctx.Process(target=_worker, args=(os.path.join(d, "init"), q))
        p.start()
        out = q.get(timeout=240)
        p.join(timeout=60)
    assert isinstance(out, dict), out
    assert out == {"sum": True, "copy": True, "allreduce": True, "graph": True}

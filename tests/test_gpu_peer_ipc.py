"""The peer-memory exchange across processes: two ranks, one process each, their
exchange buffers mapped with CUDA IPC handles traded over torch.distributed (gloo),
as in a one-process-per-GPU run.  Here both processes share GPU 0 (a functional check
of the IPC mapping, the cross-process flag release and the front-end waits; no kernel
waits on another).  Every rank must end with the same new mean, equal to world = 1
within the MPPI regrouping tolerance."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2403_11383_b200 import binding as B
    from paper_2403_11383_b200 import workloads as W
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B.load_library()
    cfg, inputs = W.config2(K=20000)
    c = B.Controller(cfg, rank=rank, world=world)
    c.set_reference(0, inputs[0]["xref"])
    handle, _ = c.peer_handle()
    handles = [None] * world
    dist.all_gather_object(handles, handle)
    c.peer_connect(handles=handles)
    d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
    d_out = torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
    means = []
    for _ in range(3):
        c.step_device(d_in.data_ptr(), d_out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        o = B.output_dict(B.sbs_output.from_buffer_copy(d_out.cpu().numpy().tobytes()), 48)
        means.append(o["mean"].copy())
    dist.barrier()
    q.put((rank, means))
    dist.barrier()
    c.close()
    dist.destroy_process_group()


def test_two_process_ipc_peer_exchange():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_11383_b200 import binding as B
    from paper_2403_11383_b200 import build
    from paper_2403_11383_b200 import workloads as W
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for a, b in zip(res[0][1], res[1][1]):
        np.testing.assert_array_equal(a, b)
    B.load_library()
    cfg, inputs = W.config2(K=20000)
    single = B.Controller(cfg)
    single.set_reference(0, inputs[0]["xref"])
    _, so = single.step(inputs)
    assert np.max(np.abs(res[0][1][0] - so[0]["mean"])) <= 1e-5 * max(np.max(np.abs(so[0]["mean"])), 1.0)

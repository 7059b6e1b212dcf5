"""World-size-2 CPU (gloo) tests of the multi-rank host logic.

On the GPU path every rank runs the FSE for the (frame, tile) units it owns
(LPT on core pixels, tf_core_layout; replaces i mod n of runtime.hpp:102), packs their cores with the layout of
tf_core_layout and NCCL-gathers them to rank 0, which unpacks them.  Here the
same host-side layout and ownership are exercised over gloo; the per-tile FSE
results come from the CPU oracle (test scaffolding standing in for the GPU;
the oracle is the checker of the assembled frame as well).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

W, H, FRAMES, TILES, OVERLAP = 96, 64, 2, 5, 8
P = (8, 8, 30, 0.5, 0.8)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _frames():
    from paper_2207_00238_b200 import tframe as T
    imgs, kns = zip(*[T.synth_frame(2, f, W, H) for f in range(FRAMES)])
    return np.stack(imgs), np.stack(kns)


def _worker(rank, world, port, q):
    import ctypes as C
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle as O
    from paper_2207_00238_b200 import _native as N
    from paper_2207_00238_b200 import tframe as T

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img, kn = _frames()
        n = FRAMES * TILES
        cores = (N.tf_rect * n)()
        fr = np.zeros(n, np.int32)
        own = np.zeros(n, np.int32)
        offs = np.zeros(n, np.int64)
        pb = np.zeros(world, np.int64)
        N.check(N.lib().tf_core_layout(W, H, FRAMES, TILES, world, cores, fr.ctypes.data,
                                       own.ctypes.data, offs.ctypes.data, pb.ctypes.data))
        # this rank's payload: cores of the tiles it owns, FSE on the halo
        payload = np.zeros(int(pb.max()), np.uint8)
        for t in range(n):
            if own[t] != rank:
                continue
            c = cores[t]
            e = T.expand(T.Rect(c.x, c.y, c.w, c.h), OVERLAP, W, H)
            h = e.halo
            sub = O.fse_lite(img[fr[t], h.y:h.y + h.h, h.x:h.x + h.w],
                             kn[fr[t], h.y:h.y + h.h, h.x:h.x + h.w], *P)
            core = sub[c.y - h.y:c.y - h.y + c.h, c.x - h.x:c.x - h.x + c.w]
            payload[offs[t]:offs[t] + c.w * c.h] = core.reshape(-1)
        got = [torch.zeros(int(pb.max()), dtype=torch.uint8) for _ in range(world)] if rank == 0 else None
        dist.gather(torch.from_numpy(payload), got, dst=0)
        if rank == 0:
            out = np.zeros_like(img)
            for t in range(n):
                c = cores[t]
                buf = got[own[t]].numpy()
                out[fr[t], c.y:c.y + c.h, c.x:c.x + c.w] = buf[offs[t]:offs[t] + c.w * c.h].reshape(c.h, c.w)
            want, _ = O.tiled(img, kn, TILES, OVERLAP, *P)
            q.put(("ok", int((out != want).sum())))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_rank_core_gather_reassembles_the_frame():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = q.get(timeout=10)
    assert res == ("ok", 0), res
    assert all(p.exitcode == 0 for p in procs)


def test_ownership_is_independent_of_world_size():
    """The assembled output must not depend on the rank count (runtime.hpp:71-74):
    every (frame, tile) unit is owned exactly once for any n."""
    from paper_2207_00238_b200 import _native as N
    n = FRAMES * TILES
    for world in (1, 2, 3, 8):
        own = np.zeros(n, np.int32)
        N.check(N.lib().tf_core_layout(W, H, FRAMES, TILES, world, None, None, own.ctypes.data, None, None))
        assert np.bincount(own, minlength=world).sum() == n
        assert sorted(set(own.tolist())) == list(range(min(world, n)))

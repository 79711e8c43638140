"""NCCL entry points of the C ABI (mvamg_comm_*, mvamg_halo_exchange,
mvamg_allreduce_sum_f64) on one GPU: a one-rank communicator, an allreduce
(identity over one rank) and a grouped send/receive to itself.  The
multi-rank exchange logic is covered under gloo on CPU (tests/test_distributed.py)."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_comm_one_rank_allreduce_and_self_exchange():
    import torch

    from paper_1907_04417_b200 import _lib
    from paper_1907_04417_b200.device import ptr, stream_handle

    L = _lib.load()
    uid = ctypes.create_string_buffer(128)
    _lib.check(L.mvamg_comm_unique_id(uid), "comm_unique_id")
    comm = ctypes.c_void_p()
    _lib.check(L.mvamg_comm_init(ctypes.byref(comm), 0, 1, uid), "comm_init")
    try:
        s = stream_handle()
        v = torch.arange(7, dtype=torch.float64, device="cuda")
        _lib.check(L.mvamg_allreduce_sum_f64(comm, ptr(v), 7, s), "allreduce")
        torch.cuda.synchronize()
        assert np.array_equal(v.cpu().numpy(), np.arange(7.0))
        src = torch.from_numpy(np.random.default_rng(0).standard_normal(100)).cuda()
        dst = torch.zeros(100, dtype=torch.float64, device="cuda")
        peers = (ctypes.c_int * 1)(0)
        sbuf = (ctypes.c_void_p * 1)(src.data_ptr())
        rbuf = (ctypes.c_void_p * 1)(dst.data_ptr())
        cnt = (ctypes.c_longlong * 1)(100)
        _lib.check(L.mvamg_halo_exchange(comm, 1, peers, sbuf, cnt, 1, peers, rbuf, cnt, s), "halo_exchange")
        torch.cuda.synchronize()
        assert torch.equal(src, dst)
        with pytest.raises(ValueError):
            _lib.check(L.mvamg_comm_init(ctypes.byref(ctypes.c_void_p()), 1, 1, uid), "comm_init")
    finally:
        L.mvamg_comm_destroy(comm)

"""Two-rank NCCL path of SURVEY §8e on GPUs: each rank runs the parallel template on its own
(b, KV-group) shard through the C ABI, the outputs are all-gathered over NCCL, and the gathered
global O equals a single-process run of the whole batch.  Skipped with fewer than two GPUs (the
gloo world-2 tests cover the host logic on CPU)."""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    import paper_2502_15349_b200 as af
    from paper_2502_15349_b200.shard import gather_batch_rows, shard_units
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    B, H, HKV, S, D = 2, 4, 2, 256, 128
    spec = af.with_causal_mask(af.builtin("softmax", batch=B, heads=H, heads_kv=HKV, seq=S,
                                          d_qk=D, d_v=D))
    shard = shard_units(B * world, HKV, world, rank)
    b_lo = shard.units[0] // HKV
    g = torch.Generator(device="cuda").manual_seed(7)
    full_in = {n: (torch.rand(B * world, h, S, D, device="cuda", generator=g) * 2 - 1)
               .to(torch.bfloat16) for n, h in (("q", H), ("k", HKV), ("v", HKV))}
    mine = {n: t[b_lo: b_lo + B].contiguous() for n, t in full_in.items()}
    o, lse = af.parallel_forward(spec, mine)
    o_all, lse_all = gather_batch_rows([o, lse], world)
    spec_all = af.with_causal_mask(af.builtin("softmax", batch=B * world, heads=H, heads_kv=HKV,
                                              seq=S, d_qk=D, d_v=D))
    o_ref, lse_ref = af.parallel_forward(spec_all, full_in)
    q.put((rank, bool(torch.equal(o_all, o_ref)), bool(torch.equal(lse_all, lse_ref))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs")
def test_nccl_world2_shards_gather_to_the_single_process_result():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(a and b for _, a, b in res), res

"""World-2 NCCL run of the table-sharded search: one process per GPU
(torch.multiprocessing, NCCL), rows block-distributed, tables round-robin,
the occurrence filter's degree / mark reductions over NCCL — triplets and
every SearchStats field byte-equal to the 1-GPU search of the same station.
Skipped on boxes with fewer than two GPUs (the driver's GPU tier has one;
tests/test_sharded_cpu.py covers the protocol with gloo ranks on CPU)."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")

pytestmark = [
    pytest.mark.gpu,
    pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                       reason="needs two GPUs"),
]

N = 40_000


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cfg(occ):
    from paper_1803_09835_b200 import lsh_search as ls
    return ls.SearchConfig(tables=100, hash_funcs=4, min_matches=5, seed=0, partitions=1,
                           occurrence_threshold=occ)


def _worker(rank, world, port, occ, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device(f"cuda:{rank}"))
    try:
        from paper_1803_09835_b200 import minmax_hash as mh
        from paper_1803_09835_b200 import sharded as sh
        from paper_1803_09835_b200 import workloads
        bits, _ = workloads.cfg1_bits_torch(n=N, seed=3, device=f"cuda:{rank}", group_frac=1 / 200)
        a, b, s = sh.row_block(N, world, rank)
        blk = bits[a:b]
        if b - a < s:
            blk = torch.cat([blk, blk[:1].expand(s - (b - a), -1)])
        mapping = mh.gen_hash_mapping(4096, 100, 4, 0)
        trip, st, _ = sh.search_bits_sharded(blk.contiguous(), N, _cfg(occ), mapping, 0)
        if rank == 0:
            q.put((trip.cpu().numpy().tobytes(), st.to_dict()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("occ", [None, 60 / N])
def test_nccl_world2_equals_one_gpu(occ):
    import torch.multiprocessing as mp
    from paper_1803_09835_b200 import lsh_search as ls
    from paper_1803_09835_b200 import minmax_hash as mh
    from paper_1803_09835_b200 import workloads
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, occ, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    got_trip, got_stats = q.get()
    bits, _ = workloads.cfg1_bits_torch(n=N, seed=3, device="cuda:0", group_frac=1 / 200)
    mapping = mh.gen_hash_mapping(4096, 100, 4, 0)
    keys, rkeys, tags, _ = ls.signatures_for_search(bits, mapping)
    trip, st, _ = ls.run_search(keys, rkeys, tags, N, 100, _cfg(occ), 0)
    assert got_trip == trip.cpu().numpy().tobytes()
    assert got_stats == st.to_dict()

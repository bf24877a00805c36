"""N>1 host logic on CPU: world_size-2 gloo processes build the shard
pointer tables (IPC primitives faked: handles encode the owner's address)."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_04398_b200.dist import ShardGroup

    class Fake(ShardGroup):
        next_addr = 0x10000 * (rank + 1)

        def _alloc(self, nbytes):
            a = Fake.next_addr
            Fake.next_addr += (nbytes + 255) // 256 * 256
            return a

        def _ipc_handle(self, ptr):
            return ptr.to_bytes(8, "little") + bytes(56)

        def _ipc_open(self, handle):
            return 0x7f00_0000_0000 + int.from_bytes(handle[:8], "little")  # "mapped" address

    g = Fake.from_torch_distributed()
    g.__class__ = Fake
    G, N = 4, 16
    sizes = {"partial": 1000, "xin": 512}
    peer, local = g.peer_tables(G, N, sizes)
    q.put((rank, peer, local))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_peer_tables_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict((r, (peer, local)) for r, peer, local in (q.get(timeout=100) for _ in range(2)))
    for p in ps:
        p.join(timeout=30)
        assert p.exitcode == 0
    L = 2
    for r in (0, 1):
        peer, local = got[r]
        for name, size in (("partial", 1000), ("xin", 512)):
            for gs in range(4):
                owner = gs // L
                owner_base = got[owner][1][name]
                want = owner_base + (gs % L) * size
                if owner != r:
                    want += 0x7f00_0000_0000            # mapped through the fake IPC
                assert peer[name][gs] == want, (r, name, gs)
        # one counts / signal pad per process, shared by its shards
        assert peer["counts"][0] == peer["counts"][1] and peer["counts"][2] == peer["counts"][3]
        assert peer["signal"][r * L] == local["signal"]

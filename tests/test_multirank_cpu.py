"""CPU tests of the multi-GPU host logic with a real 2-process torch.distributed (gloo) group:
* the count-balanced Morton splitters (p2p_partition_splitters, the function the collective plan build uses)
  computed independently on each rank from an all-reduced supercell histogram agree bit for bit across ranks,
  cover the key space with contiguous ranges and balance the particle counts;
* the NCCL unique-id bootstrap: rank 0's 128 id bytes arrive unchanged on every rank (the broadcast bench.py
  performs before p2p_comm_create).
Keys come from the oracle (test infrastructure); the library is only asked for the splitters."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import p2p_inputs as G
        import paper_2511_21535_b200 as P
        inp = G.plummer(40000, 32, seed=11)
        mine = np.arange(inp.n)[rank::world]             # an arbitrary (non-spatial) initial distribution
        ib = oracle.bin_positions(inp.pos[mine], inp.h, inp.lo, inp.nbox)
        nb = oracle.bits_per_dim(inp.nbox)
        keys = np.array([oracle.morton(3, nb, c) for c in ib], dtype=np.uint64)
        key_bits = 3 * nb
        sc_bits = min(key_bits, 12)
        shift = key_bits - sc_bits
        hist = np.bincount((keys >> shift).astype(np.int64), minlength=1 << sc_bits).astype(np.int64)
        t = torch.from_numpy(hist)
        dist.all_reduce(t)
        ghist = t.numpy().astype(np.uint64)
        spl = P.p2p_partition_splitters(ghist, shift, key_bits, world)
        allspl = [torch.zeros(world + 1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allspl, torch.from_numpy(spl.astype(np.int64)))
        # NCCL unique id bootstrap over the CPU group
        idb = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            try:
                idb = torch.frombuffer(bytearray(P.p2p_comm_unique_id()), dtype=torch.uint8).clone()
            except Exception:  # noqa: BLE001 -- no NCCL bootstrap possible on this host
                idb = torch.full((128,), 7, dtype=torch.uint8)
        dist.broadcast(idb, 0)
        ids = [torch.zeros(128, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(ids, idb)
        # global key list for the balance check
        allkeys = [torch.zeros(0)] * world
        kk = torch.from_numpy(keys.astype(np.int64))
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([kk.numel()]))
        mx = int(max(s.item() for s in sizes))
        pad = torch.full((mx,), -1, dtype=torch.int64)
        pad[:kk.numel()] = kk
        allkeys = [torch.zeros(mx, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allkeys, pad)
        q.put((rank, [a.numpy() for a in allspl], [i.numpy() for i in ids],
               np.concatenate([a.numpy()[a.numpy() >= 0] for a in allkeys]), key_bits, int(ghist.max())))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001 -- reported to the parent
        q.put((rank, repr(e)))


def test_splitters_and_bootstrap_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert len(r) > 2, r
    rank, spls, ids, keys, key_bits, maxbin = res[0]
    for r in res:
        # every rank computed the same splitters and received the same id bytes
        for s in r[1]:
            assert np.array_equal(s, spls[0])
        for i in r[2]:
            assert np.array_equal(i, ids[0])
    spl = spls[0]
    assert spl[0] == 0 and spl[-1] == 1 << key_bits and np.all(np.diff(spl) >= 0)
    counts = [np.count_nonzero((keys >= spl[r]) & (keys < spl[r + 1])) for r in range(world)]
    assert sum(counts) == keys.size
    # balance within one supercell of the ideal split
    assert max(abs(c - keys.size / world) for c in counts) <= maxbin

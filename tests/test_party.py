"""Three-host deployment: one process per party, every
protocol round a real message on the P_i -> P_{i+1} ring (transport.py:374-475,
rss.py:371-412).

* CPU (gloo, 3 ranks): the ring's two message directions and the per-party
  message log;
* GPU (gloo between 3 processes sharing cuda:0; NCCL between GPUs in a real
  deployment): infer_batch (infer.py:20-35) with each party holding only its
  own pairs and its own dealt material bank -> revealed predictions equal the
  plaintext walk, the returned pairs are replicated, and each party sends
  exactly the bytes / rounds of the reference's transcript (ledger)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ring_worker(rank, port, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_2305_00645_b200.party import RingComm

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=3)
    party = rank + 1
    comm = RingComm(party)
    a = comm.to_next(torch.full((5,), 10 * party, dtype=torch.int64))  # from prev
    b = comm.to_prev(torch.full((3,), 7 * party, dtype=torch.uint8))  # from next
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), a=a.numpy(), b=b.numpy(),
             log=np.array(comm.transcript.records, dtype=object))
    dist.barrier()
    dist.destroy_process_group()


def test_ring_messages_cpu(tmp_path):
    mp.spawn(_ring_worker, args=(_port(), str(tmp_path)), nprocs=3, join=True)
    for p in (1, 2, 3):
        z = np.load(tmp_path / f"r{p - 1}.npz", allow_pickle=True)
        prev, nxt = (p + 1) % 3 + 1, p % 3 + 1
        assert (z["a"] == 10 * prev).all() and (z["b"] == 7 * nxt).all()
        assert [tuple(r) for r in z["log"]] == [(1, p, nxt, 40, "msg"), (2, p, prev, 3, "msg")]


def _infer_worker(rank, port, out_dir, depth, nq, nf):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle import shadow
    from paper_2305_00645_b200.material import generate_material, inference_needs
    from paper_2305_00645_b200.party import HostParty, RingComm
    from paper_2305_00645_b200.seeds import SeedSetup, derive_seed
    from conftest import share

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=3)
    torch.cuda.set_device(0)
    party = rank + 1
    rng = np.random.default_rng(5)  # every party draws the same dealing; each keeps only its pairs
    Tv, _ = shadow.random_tree(rng, depth, nf + 1)
    q = rng.integers(0, 2, (nq, nf), dtype=np.uint8)
    Tc, Qc = share(Tv, rng), share(q, rng)
    mine = [party - 1, party % 3]
    dev = lambda c: torch.from_numpy(np.ascontiguousarray(c[mine]).view(np.int64)).cuda()  # noqa: E731
    setup = SeedSetup.from_master(b"\x33" * 16)
    bank = generate_material(inference_needs(nq, depth, nf + 1), derive_seed(setup.master, "deal/material"))[party - 1]
    hp = HostParty(party, RingComm(party), setup.pair_seeds[party], setup.pair_seeds[(party + 1) % 3 + 1], bank)
    out = hp.infer_batch(dev(Tc), depth, dev(Qc))
    torch.cuda.synchronize()
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), out=out.cpu().numpy().view(np.uint64),
             sent=sum(r[3] for r in hp.comm.transcript.records), rounds=hp.comm.round_no,
             want=shadow.plaintext_infer(Tv, depth, q))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("depth,nq,nf", [(3, 257, 5), (7, 1000, 13)])
def test_three_host_inference_over_the_ring(tmp_path, depth, nq, nf):
    from paper_2305_00645_b200 import ledger

    mp.spawn(_infer_worker, args=(_port(), str(tmp_path), depth, nq, nf), nprocs=3, join=True)
    z = [np.load(tmp_path / f"r{r}.npz") for r in range(3)]
    pairs = [x["out"] for x in z]
    for p in range(3):  # replicated: party p's hi is party p+1's lo
        assert np.array_equal(pairs[p][1], pairs[(p + 1) % 3][0])
    preds = pairs[0][0] + pairs[1][0] + pairs[2][0]
    assert np.array_equal(preds, z[0]["want"])
    ref = ledger.infer_metrics(nq, nf, depth, lane_limit=None)
    for p in range(3):
        assert int(z[p]["rounds"]) == ref.rounds == 18 * depth
        assert int(z[p]["sent"]) == ref.sent_by_party(p + 1)


def _dir_worker(rank, port, base, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_2305_00645_b200.party import RingComm, infer_party_dir

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=3)
    torch.cuda.set_device(0)
    out = infer_party_dir(base, rank + 1, RingComm(rank + 1))
    np.save(os.path.join(out_dir, f"r{rank}.npy"), out.cpu().numpy().view(np.uint64))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_three_host_inference_from_party_directories(tmp_path):
    """Each process reads only its own partyN/ directory of a dealt inference
    (queries and tree shares, seeds, material.bin) -- the reference's
    deal-then-serve flow (cli.py:344-400, 590-615)."""
    import json

    from oracle import shadow
    from paper_2305_00645_b200.material import generate_material, inference_needs
    from paper_2305_00645_b200.seeds import SeedSetup, derive_seed
    from paper_2305_00645_b200.shares import RING64, pairs_from_components, write_share_file
    from conftest import share

    depth, nq, nf = 4, 300, 7
    rng = np.random.default_rng(8)
    Tv, _ = shadow.random_tree(rng, depth, nf + 1)
    q = rng.integers(0, 2, (nq, nf), dtype=np.uint8)
    setup = SeedSetup.from_master(b"\x44" * 16)
    banks = generate_material(inference_needs(nq, depth, nf + 1), derive_seed(setup.master, "deal/material"))
    base = tmp_path / "deal"
    Tp, Qp = pairs_from_components(share(Tv, rng)), pairs_from_components(share(q.reshape(-1), rng))
    for p in (1, 2, 3):
        d = base / f"party{p}"
        d.mkdir(parents=True)
        (d / "seeds.json").write_text(json.dumps({"party": p, "pair_next": setup.pair_seeds[p].hex(),
                                                  "pair_prev": setup.pair_seeds[(p + 1) % 3 + 1].hex()}))
        write_share_file(str(d / "tree_T.shr"), *Tp[p - 1], RING64, p)
        write_share_file(str(d / "queries.shr"), *Qp[p - 1], RING64, p)
        banks[p - 1].to_file(str(d / "material.bin"))
    (base / "meta.json").write_text(json.dumps({"kind": "infer", "n_rows": nq, "n_columns": nf + 1, "depth": depth}))
    mp.spawn(_dir_worker, args=(_port(), str(base), str(tmp_path)), nprocs=3, join=True)
    outs = [np.load(tmp_path / f"r{r}.npy") for r in range(3)]
    assert np.array_equal(outs[0][0] + outs[1][0] + outs[2][0], shadow.plaintext_infer(Tv, depth, q))

"""Three-host deployment: one party per rank, real messages on the ring.

SURVEY.md 8(f)4.  The co-resident engine (engine.py) holds all three
parties' shares on one device, so an open or a reshare is an identity.  Here
each party is its own process (a rank of a 3-rank torch.distributed group:
NCCL between GPUs, or gloo), holds only its replicated pair (lo, hi) =
(c_{p-1}, c_p) of every shared vector (rss.py:1-9), and every protocol round
is an actual message on the P_i -> P_{i+1} ring (the reference's TcpChannel
mesh, transport.py:374-475, with the message pattern of rss.py:371-412):

* open (open_a / open_bits): send lo to next, receive prev's lo;
* mul / and: send the fresh local z_i to prev, receive z_{i+1} from next.

The local math of each round is a party-local kernel (csrc/gt_party.cu);
correlated material comes from this party's dealt OBD1 bank (material.py)
on the device, zero shares from the two pairwise keys the party holds.
``HostParty.infer_batch`` runs the reference's infer_batch (infer.py:20-35)
this way, 18 rounds per level; the per-party message log has the
reference's sizes (np.packbits byte counts for bit rounds).  Training stays
co-resident (the count of a level is N x 2^h eq lanes per round trip: a
ring deployment of it is transport-bound).
"""

from __future__ import annotations

import ctypes
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _native
from .ledger import Transcript
from .material import MaterialBank
from .seeds import philox_key

SITE_WALK_OAA, SITE_WALK_ROW = 16, 17  # gt_common.cuh op sites (walk:t)
_AND_SUBS = 6  # in-word AND tree of a 64-bit eq: 64 -> 32 -> ... -> 1
_SELECT_SUB = 8


def _op(level: int, site: int) -> int:
    return (level << 16) | site


class RingComm:
    """The three-party ring over torch.distributed.  `ranks[p - 1]` is party
    p's rank in `group` (default: rank r = party r + 1)."""

    def __init__(self, party: int, group=None, ranks: Optional[Sequence[int]] = None):
        import torch.distributed as dist

        if party not in (1, 2, 3):
            raise ValueError("party must be 1, 2 or 3")
        self.dist, self.group, self.party = dist, group, party
        self.ranks = list(ranks) if ranks is not None else [0, 1, 2]
        self.next = self.ranks[party % 3]
        self.prev = self.ranks[(party + 1) % 3]
        self.nccl = dist.get_backend(group) == "nccl"
        self.transcript = Transcript()
        self.round_no = 0
        self.tag = "msg"

    def _xchg(self, t, to: int, frm: int, receiver_party: int):
        import torch

        dist = self.dist
        self.round_no += 1
        nbytes = t.numel() * t.element_size()
        self.transcript.append(self.round_no, self.party, receiver_party, nbytes, self.tag)
        if self.nccl:  # device buffers straight over NVLink / the network
            buf = torch.empty_like(t)
            reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, t.contiguous(), to, self.group),
                                           dist.P2POp(dist.irecv, buf, frm, self.group)])
            for r in reqs:
                r.wait()
            return buf
        tc = t.contiguous().cpu()  # gloo moves host buffers
        bc = torch.empty_like(tc)
        r1 = dist.isend(tc, to, self.group)
        r2 = dist.irecv(bc, frm, self.group)
        r1.wait()
        r2.wait()
        return bc.to(t.device)

    def to_next(self, t):
        """open: my lo goes to next, prev's lo comes back."""
        return self._xchg(t, self.next, self.prev, self.party % 3 + 1)

    def to_prev(self, t):
        """reshare: my z goes to prev, next's z comes back."""
        return self._xchg(t, self.prev, self.next, (self.party + 1) % 3 + 1)


class HostParty:
    """One party of a three-host run: its pairwise keys (pair_next shared with
    the next party, pair_prev with the previous one -- the reference's
    partyN/seeds.json, cli.py:281-300), its dealt material bank and the ring."""

    def __init__(self, party: int, comm: RingComm, pair_next: bytes, pair_prev: bytes, bank: MaterialBank,
                 device=None):
        torch = _native.require_cuda()
        self.lib = _native.load()
        self.party, self.comm = party, comm
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        k = _native.gt_keys()
        k.pair[party - 1].k0, k.pair[party - 1].k1 = philox_key(pair_next)
        k.pair[(party + 1) % 3].k0, k.pair[(party + 1) % 3].k1 = philox_key(pair_prev)
        self.keys = k
        self.material: Dict[tuple, List] = {}
        self.cursor: Dict[tuple, int] = {}
        for key, arrays in bank.sections.items():  # field pairs -> [2, count] device tensors
            fields = []
            for f in range(0, len(arrays), 2):
                pair = np.stack([arrays[f], arrays[f + 1]])
                if pair.dtype == np.uint8:
                    fields.append(torch.from_numpy(pair).to(self.device))
                else:
                    fields.append(torch.from_numpy(pair.astype(np.uint64).view(np.int64)).to(self.device))
            self.material[key] = fields
            self.cursor[key] = 0

    # -- plumbing ---------------------------------------------------------------
    def _stream(self):
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _call(self, fn, *args):
        _native.check(getattr(self.lib, fn)(*args, self._stream()))

    def _take(self, key: tuple, n: int):
        from .material import MaterialError

        have = self.material.get(key)
        at = self.cursor.get(key, 0)
        if have is None or have[0].shape[1] - at < n:
            raise MaterialError(f"material exhausted for {key}: requested {n}, have "
                                f"{0 if have is None else have[0].shape[1] - at}")
        self.cursor[key] = at + n
        return [f[:, at:at + n].contiguous() for f in have]

    def _new(self, *shape, dtype=None):
        import torch

        return torch.empty(shape, dtype=dtype or torch.int64, device=self.device)

    # -- protocol ---------------------------------------------------------------
    def lookup(self, idx, table, m: int, off: int, per_row: bool, op: int):
        """oaa / row_lookup (oaa.py:20-55) of one pair vector of indices
        idx [2, nq] (minus the public `off`) over m entries: eq lanes vs the
        ramp, b2a of the hits, select against zero, summed per index."""
        import torch

        nq = idx.shape[1]
        L = nq * m
        ptr = lambda t: t.data_ptr()  # noqa: E731
        kp = ctypes.addressof(self.keys)
        r, rbits = self._take(("edabit", 64), L)
        masked = self._new(2, L)
        self._call("gt_party_eq_mask", self.party, ptr(idx), nq, m, off, ptr(r), ptr(masked))
        self.comm.tag = "eq.open"
        recv = self.comm.to_next(masked[0])
        planes = self._new(2, L)
        self._call("gt_party_eq_planes", self.party, ptr(masked), ptr(recv), ptr(rbits), L, ptr(planes))
        width = 64
        for sub in range(_AND_SUBS):  # and_reduce: one ring round per level
            z = self._new(L)
            self._call("gt_party_and_half", self.party, ptr(planes), L, width, kp, op, sub, 0, ptr(z))
            width //= 2
            packed = self._new((L * width + 7) // 8, dtype=torch.uint8)
            self._call("gt_party_pack", ptr(z), L, width, ptr(packed))
            self.comm.tag = "and"
            got = self.comm.to_prev(packed)
            zn = self._new(L)
            self._call("gt_party_unpack", ptr(got), L, width, ptr(zn))
            planes = torch.stack([z, zn])
        a, bb = self._take(("dabit", 64), L)
        em = self._new(2, L)
        self._call("gt_party_b2a_mask", ptr(planes), ptr(bb), L, ptr(em))
        packed = self._new((L + 7) // 8, dtype=torch.uint8)
        self._call("gt_party_pack", ptr(em), L, 1, ptr(packed))
        self.comm.tag = "b2a.open"
        got = self.comm.to_next(packed)
        ev = self._new(L)
        self._call("gt_party_unpack", ptr(got), L, 1, ptr(ev))
        ca = self._new(2, L)
        self._call("gt_party_b2a_finish", self.party, ptr(em), ptr(ev), ptr(a), L, ptr(ca))
        z = self._new(L)
        self._call("gt_party_select_mul", self.party, ptr(ca), ptr(table), table.shape[1], 1 if per_row else 0, nq, m,
                   kp, op, _SELECT_SUB, 0, ptr(z))
        self.comm.tag = "select.mul"
        zn = self.comm.to_prev(z)
        picked = torch.stack([z, zn])
        out = self._new(2, nq)
        self._call("gt_party_lane_sum", ptr(picked), nq, m, ptr(out))
        return out

    def infer_batch(self, tree, depth: int, queries):
        """infer_batch (infer.py:20-35) on this party's pairs: tree [2, 2^H - 1]
        heap payloads, queries [2, nq, nf] -> predicted labels [2, nq]."""
        import torch

        nq, nf = queries.shape[1], queries.shape[2]
        rows = queries.reshape(2, nq * nf).contiguous()
        slot = torch.zeros((2, nq), dtype=torch.int64, device=self.device)  # const(0)
        payload = slot
        for t in range(depth):
            m, o = 1 << t, (1 << t) - 1
            level = tree[:, o:o + m].contiguous()
            payload = self.lookup(slot, level, m, o, False, _op(t, SITE_WALK_OAA))
            branch = self.lookup(payload, rows, nf, 0, True, _op(t, SITE_WALK_ROW))
            _native.check(self.lib.gt_party_slot_step(self.party, slot.data_ptr(), branch.data_ptr(), nq,
                                                      self._stream()))
        return payload


def load_party_pair(path: str, device, shape=None):
    """This party's own OBS1 share file (rss.py:452-481) -> its pair [2, ...]
    on the device (the three-host counterpart of material.load_share_files)."""
    import torch

    from .shares import read_share_file

    lo, hi, _, _ = read_share_file(path)
    pair = np.stack([lo, hi]).astype(np.uint64)
    if shape is not None:
        pair = pair.reshape((2,) + tuple(shape))
    return torch.from_numpy(np.ascontiguousarray(pair).view(np.int64)).to(device)


def infer_party_dir(base: str, party: int, comm: RingComm, device=None):
    """One party's side of a dealt inference (the reference's _infer_tcp,
    cli.py:590-615): reads ONLY partyN/ of the deal directory -- its seeds
    (pair_next / pair_prev), its queries.shr and tree_T.shr pairs, its
    material.bin -- and walks the tree over the ring.  Returns its pair of the
    predicted labels [2, nq]."""
    import json
    import os

    d = os.path.join(base, f"party{party}")
    with open(os.path.join(base, "meta.json")) as fh:
        meta = json.load(fh)
    with open(os.path.join(d, "seeds.json")) as fh:
        seeds = json.load(fh)
    if int(seeds["party"]) != party:
        raise ValueError(f"{d} holds party {seeds['party']}'s seeds")
    torch = _native.require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    n, ncol, depth = int(meta["n_rows"]), int(meta["n_columns"]), int(meta["depth"])
    hp = HostParty(party, comm, bytes.fromhex(seeds["pair_next"]), bytes.fromhex(seeds["pair_prev"]),
                   MaterialBank.from_file(os.path.join(d, "material.bin")), dev)
    Q = load_party_pair(os.path.join(d, "queries.shr"), dev, (n, ncol - 1))
    T = load_party_pair(os.path.join(d, "tree_T.shr"), dev)
    return hp.infer_batch(T, depth, Q)

"""Candidate sharding across GPUs (one process per GPU, torch.distributed).

Every t_max candidate's DP is independent (planner.py:526-531),
so a batch of candidates is dealt across ranks in contiguous blocks of 128
candidates, back and forth (0..W-1, W-1..0, ...): blocks keep the DP's
candidate groups t_max-contiguous (tight lane bounds), and the boustrophedon
deal balances the ranks as the activated span count grows with t_max.
Each rank builds the same K1 tables locally (microseconds; cheaper than a
broadcast).  The only exchange steps are

  * all_gather of per-candidate (T*, best_s, dp_states) when every rank must
    replay the reference's pruning decisions identically (search()), and
  * an allreduce-argmin of (T*, index) -- two 8-byte MIN all-reduces, since
    non-negative IEEE doubles order like their bit patterns -- that picks the
    global winner of a full-pool sweep (the merge of planner.py:535-541).

With the NCCL backend the collectives run on device tensors over NVLink /
NVSwitch; the same code runs on gloo (CPU tensors) for the CPU test suite.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

_I64_MAX = np.iinfo(np.int64).max


class PoolSharding:
    """min_shard: batches smaller than this are evaluated whole on every rank
    (identical results, no collective) -- a small probe batch does not fill
    one GPU, so splitting it only adds an all_gather to its latency."""

    MIN_SHARD = 1024

    def __init__(self, group=None, min_shard: int | None = None):
        self.min_shard = self.MIN_SHARD if min_shard is None else int(min_shard)
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed is not initialised")
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        self.collective_calls = 0

    @property
    def device(self) -> torch.device:
        if self.backend == "nccl":
            return torch.device("cuda", torch.cuda.current_device())
        return torch.device("cpu")

    BLOCK = 128  # candidates per contiguous block (the widest DP candidate group)

    def shard_positions(self, n: int) -> np.ndarray:
        """Positions of this rank's share of n sorted candidates: contiguous
        blocks of BLOCK dealt round-robin.  Candidates of a block have
        neighbouring t_max, so a DP candidate group (32-128 lanes) keeps tight
        lane bounds and finite ranges (a strided share spreads each group
        over a W-times wider t_max range: D3 at 4 GPUs ran 3.1x instead of
        ~4x); dealing the blocks back and forth keeps the ranks balanced as
        the per-candidate work grows with t_max."""
        return self._positions(n, self.rank)

    def _positions(self, n: int, rank: int) -> np.ndarray:
        # blocks aligned to the DP's candidate groups: 128 when a rank's share
        # runs at 4 candidates per lane (>= 1,024 candidates), else 64 (finer
        # deal: D1's 1,786 at 4 GPUs = 28 blocks, 7 per rank); a group never
        # straddles two blocks, which would put a t_max gap inside it
        W = self.world
        blk = self.BLOCK if n >= 1024 * W else self.BLOCK // 2
        pos = np.arange(n)
        b = pos // blk
        # boustrophedon deal (0..W-1, W-1..0, ...): work grows with t_max, so a
        # plain round-robin would always hand the last rank the larger block
        owner = np.where((b // W) % 2 == 0, b % W, W - 1 - b % W)
        return pos[owner == rank]

    def shard(self, indices):
        idx = list(indices)
        return [idx[p] for p in self.shard_positions(len(idx))]

    def _all_gather(self, local: torch.Tensor, width: int) -> torch.Tensor:
        """Gather equally padded [width, ...] tensors from every rank."""
        pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=self.device)
        pad[: local.shape[0]] = local.to(self.device)
        out = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(out, pad, group=self.group)
        self.collective_calls += 1
        return torch.stack(out).cpu()

    def evaluate_sharded(self, sweeper, pool: np.ndarray, todo, num_microbatches: int,
                         want_ftop: bool = False):
        """Evaluate pool[todo] with each rank taking todo[rank::world]; every
        rank returns the full (tstar, best_s, states) in `todo` order, plus
        F[s,1,G] per candidate when want_ftop (search_batches)."""
        todo = list(todo)
        mine = self.shard(todo)
        width = max(len(self._positions(len(todo), r)) for r in range(self.world))
        s1 = sweeper.tables.s_max + 1 if want_ftop else 0
        cols = 3 + s1
        if mine:
            res = (sweeper.evaluate(pool[mine], num_microbatches, keep_ftop=True) if want_ftop
                   else sweeper.evaluate(pool[mine], num_microbatches))
            parts = [res.tstar.view(np.int64)[:, None], res.best_s.astype(np.int64)[:, None],
                     res.states.astype(np.int64)[:, None]]
            if want_ftop:
                parts.append(np.ascontiguousarray(res.ftop).view(np.int64))
            loc = np.concatenate(parts, axis=1)
        else:
            loc = np.zeros((0, cols), dtype=np.int64)
        allv = self._all_gather(torch.from_numpy(np.ascontiguousarray(loc)), max(width, 1)).numpy()
        tstar = np.empty(len(todo))
        best_s = np.empty(len(todo), dtype=np.int64)
        states = np.empty(len(todo), dtype=np.int64)
        ftop = np.empty((len(todo), s1)) if want_ftop else None
        for r in range(self.world):
            pos = self._positions(len(todo), r)
            blk = allv[r, : len(pos)]
            tstar[pos] = blk[:, 0].view(np.float64)
            best_s[pos] = blk[:, 1]
            states[pos] = blk[:, 2]
            if want_ftop:
                ftop[pos] = np.ascontiguousarray(blk[:, 3:]).view(np.float64)
        if want_ftop:
            return tstar, best_s, states, ftop
        return tstar, best_s, states

    def positions_device(self, n: int, device) -> torch.Tensor:
        """shard_positions(n) as an int64 tensor on `device` (cached: a sweep
        of the same pool size reuses it instead of copying it again)."""
        cache = getattr(self, "_mine_cache", None)
        key = (n, self.world, str(device))
        if cache is None or cache[0] != key:
            cache = (key, torch.from_numpy(self.shard_positions(n)).to(device))
            self._mine_cache = cache
        return cache[1]

    def gather_positions(self, local: torch.Tensor, n: int) -> torch.Tensor:
        """All ranks' per-candidate rows, device to device: local [m, C] int64
        holds this rank's candidates in shard_positions(n) order; returns
        [n, C] in pool order on every rank (one all_gather of equally padded
        blocks, then a scatter by the deal's positions)."""
        key = (n, self.world)
        cache = getattr(self, "_pos_cache", None)
        if cache is None or cache[0] != key:
            pos = [self._positions(n, r) for r in range(self.world)]
            cache = (key, pos, {})
            self._pos_cache = cache
        pos, dev_idx = cache[1], cache[2]
        dev = self.device
        width = max(1, max(len(p) for p in pos))
        C = local.shape[1]
        pad = torch.zeros((width, C), dtype=local.dtype, device=dev)
        pad[: local.shape[0]] = local.to(dev)
        if self.backend == "nccl":
            out = torch.empty((self.world * width, C), dtype=local.dtype, device=dev)
            dist.all_gather_into_tensor(out, pad, group=self.group)
            out = out.view(self.world, width, C)
        else:
            parts = [torch.empty_like(pad) for _ in range(self.world)]
            dist.all_gather(parts, pad, group=self.group)
            out = torch.stack(parts)
        self.collective_calls += 1
        if dev not in dev_idx:
            sel = np.concatenate([r * width + np.arange(len(p)) for r, p in enumerate(pos)])
            dst = np.concatenate(pos)
            dev_idx[dev] = (torch.from_numpy(sel).to(dev), torch.from_numpy(dst).to(dev))
        sel, dst = dev_idx[dev]
        full = torch.empty((n, C), dtype=local.dtype, device=dev)
        full[dst] = out.reshape(-1, C)[sel]
        return full

    def allreduce_argmin_device(self, tstar: torch.Tensor, winner: torch.Tensor,
                                global_index: torch.Tensor):
        """Device-side allreduce-argmin of a sweep's local winner, no host
        synchronisation: tstar [n] float64 and winner [1] int32 as
        hapt_dp_select returns them (winner -1: nothing feasible here),
        global_index [n] int64 the candidates' pool indices.  One all_gather
        of a 16-byte (bits(T*), index) key per rank, then the lexicographic
        minimum on the device (non-negative IEEE doubles order like their
        bit patterns).  Returns (bits of the global T* [int64, I64_MAX if
        none], its pool index [int64, I64_MAX if none]) as device tensors."""
        dev = self.device
        w = winner.to(device=dev, dtype=torch.int64).reshape(1)
        ok = w >= 0
        wi = w.clamp(min=0)
        big = torch.full((1,), _I64_MAX, dtype=torch.int64, device=dev)
        bits = torch.where(ok, tstar.to(dev).view(torch.int64)[wi], big)
        gi = torch.where(ok, global_index.to(dev)[wi], big)
        loc = torch.cat([bits, gi]).reshape(1, 2)
        if self.backend == "nccl":
            out = torch.empty((self.world, 2), dtype=torch.int64, device=dev)
            dist.all_gather_into_tensor(out, loc, group=self.group)
        else:
            parts = [torch.empty_like(loc) for _ in range(self.world)]
            dist.all_gather(parts, loc, group=self.group)
            out = torch.cat(parts)
        self.collective_calls += 1
        gbits = out[:, 0].min()
        gidx = torch.where(out[:, 0] == gbits, out[:, 1], big.expand(self.world)).min()
        return gbits, gidx

    def allreduce_argmin(self, tstar: float, index: int):
        """Global lexicographic min of (T*, index) over ranks; (inf, -1) if
        no rank has a feasible candidate.  Two MIN all-reduces of 8 bytes."""
        feas = index >= 0 and np.isfinite(tstar)
        bits = np.array([tstar], dtype=np.float64).view(np.int64)[0] if feas else _I64_MAX
        t = torch.tensor([bits], dtype=torch.int64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        gbits = int(t.item())
        mine = index if feas and bits == gbits else _I64_MAX
        i = torch.tensor([mine], dtype=torch.int64, device=self.device)
        dist.all_reduce(i, op=dist.ReduceOp.MIN, group=self.group)
        self.collective_calls += 2
        gidx = int(i.item())
        if gbits == _I64_MAX:
            return float("inf"), -1
        return float(np.array([gbits], dtype=np.int64).view(np.float64)[0]), gidx

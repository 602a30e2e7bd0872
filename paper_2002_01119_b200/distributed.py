"""Multi-GPU layouts of the learner-averaging step.

One process per GPU; ``torch.distributed`` is plumbing only (handle exchange,
a step barrier, and the D1D all-reduce).  Two layouts:

* :class:`CoordinateShards` — rank g owns a column stripe of all L learners.
  Rows of W are independent (``(W @ T)[r, :]`` only reads row r) and every
  rank derives the same permutation from the shared seed, so
  there is no data-path communication at all.
* :class:`LearnerShardedRing` / :class:`LearnerShardedD1D` — rank g owns
  learners [row0, row0 + Lg) (north-star (d)).  The ring step pulls the
  neighbour rows it needs from the peers' HBM over NVLink *inside* the fused
  kernel (CUDA IPC mappings, ``rm_ring_mix_sgd_sharded_*``); D1D reduces local
  column sums with an NCCL all-reduce pipelined against the local kernels.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib, mixing, seeding


def balanced_split(n: int, parts: int) -> list[tuple[int, int]]:
    """[begin, end) of `parts` contiguous ranges covering range(n); the first
    n % parts ranges get one extra element."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    base, extra = divmod(n, parts)
    out, b = [], 0
    for p in range(parts):
        e = b + base + (1 if p < extra else 0)
        out.append((b, e))
        b = e
    return out


@dataclass(frozen=True)
class ShardLayout:
    """Contiguous ownership of L learners by `world` ranks."""

    L: int
    world: int

    @property
    def bounds(self) -> list[tuple[int, int]]:
        return balanced_split(self.L, self.world)

    def rows(self, rank: int) -> tuple[int, int]:
        return self.bounds[rank]

    def owner(self, learner: int) -> int:
        for r, (b, e) in enumerate(self.bounds):
            if b <= learner < e:
                return r
        raise ValueError(f"learner {learner} out of range")

    def local_index(self, learner: int) -> int:
        return learner - self.bounds[self.owner(learner)][0]


def d1d_numpy_chains(L: int, world: int, multicast_reduce: bool = False) -> int:
    """Chains per rank of the numpy-order learner-sharded D1D (rm_set_d1d_numpy_order), or 0
    where it does not apply: numpy's non-recursive pairwise mean needs 8 <= L <= 128 with
    L % 8 == 0, the eight chains must split evenly (world 1, 2, 4 or 8), and an in-switch
    (or NCCL) reduction of more than two ranks has no specified order.
    RINGMIX_D1D_NUMPY_ORDER=0 turns it off."""
    if os.environ.get("RINGMIX_D1D_NUMPY_ORDER", "1") == "0":
        return 0
    if L % 8 or not 8 <= L <= 128 or world not in (1, 2, 4, 8):
        return 0
    if multicast_reduce and world > 2:
        return 0
    return 8 // world


def d1d_learners(L: int, world: int, rank: int, chains: int) -> list[int]:
    """Global learner ids of `rank`'s local rows: with numpy-order chains, the learners of
    numpy's pairwise chains [rank * chains, (rank + 1) * chains) in ascending order
    (local row i = learner (i // chains) * 8 + rank * chains + i % chains); else the
    contiguous block of ShardLayout."""
    if chains:
        return [(i // chains) * 8 + rank * chains + i % chains for i in range(L // world)]
    b, e = ShardLayout(L, world).bounds[rank]
    return list(range(b, e))


class _NumpyOrder:
    """Scope of rm_set_d1d_numpy_order for the calling thread's launches."""

    def __init__(self, chains: int):
        self.chains = chains

    def __enter__(self):
        if self.chains:
            _lib.check(_lib.load().rm_set_d1d_numpy_order(self.chains), "rm_set_d1d_numpy_order")

    def __exit__(self, *exc):
        if self.chains:
            _lib.load().rm_set_d1d_numpy_order(0)


class _ShardStreams:
    """Scope of rm_set_shard_streams: the generator draws the numpy-order learner set
    (runs of `chains` learners every 8) for the calling thread's launches."""

    def __init__(self, chains: int):
        self.chains = chains

    def __enter__(self):
        if self.chains:
            _lib.check(_lib.load().rm_set_shard_streams(self.chains, 8), "rm_set_shard_streams")

    def __exit__(self, *exc):
        if self.chains:
            _lib.load().rm_set_shard_streams(0, 0)


def plan_reference(left, right, row0: int, Lg: int):
    """Host restatement of rm_shard_plan: (remote ids, staged triples) for the
    rank owning [row0, row0+Lg).  Used by the tests to check the device planner."""
    rem: list[int] = []

    def staged(x: int) -> int:
        if row0 <= x < row0 + Lg:
            return x - row0
        if x not in rem:
            rem.append(x)
        return Lg + rem.index(x)

    tri = []
    for j in range(Lg):
        g = row0 + j
        a, b, c = sorted((int(left[g]), g, int(right[g])))
        tri.append((staged(a), staged(b), staged(c), j))
    return rem, tri


def exchange_objects(obj, group=None) -> list:
    """all_gather_object wrapper (gloo or NCCL)."""
    world = dist.get_world_size(group)
    out = [None] * world
    dist.all_gather_object(out, obj, group=group)
    return out


# ----------------------------------------------------------------------------
# coordinate sharding
# ----------------------------------------------------------------------------

@dataclass(frozen=True)
class CoordinateShards:
    """Rank `rank` of `world` owns columns [c0, c1) of all L learners."""

    d: int
    world: int
    rank: int

    @property
    def columns(self) -> tuple[int, int]:
        return balanced_split(self.d, self.world)[self.rank]

    @property
    def width(self) -> int:
        c0, c1 = self.columns
        return c1 - c0


# ----------------------------------------------------------------------------
# learner sharding: IPC-mapped peer rows
# ----------------------------------------------------------------------------

class PeerMappedBuffers:
    """Export local device buffers with CUDA IPC, import every peer's, and return
    per-buffer base addresses for all ranks (own address for the local rank)."""

    def __init__(self, tensors: list[torch.Tensor], group=None):
        lib = _lib.load()
        hsz = lib.rm_ipc_handle_size()
        blobs = []
        for t in tensors:
            h = (ctypes.c_ubyte * hsz)()
            off = ctypes.c_uint64(0)
            _lib.check(lib.rm_ipc_get_handle(t.data_ptr(), ctypes.addressof(h),
                                             ctypes.addressof(off)), "rm_ipc_get_handle")
            blobs.append((bytes(h), int(off.value)))
        allb = exchange_objects(blobs, group)
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._opened: list[int] = []
        self.bases: list[list[int]] = []   # [rank][buffer] -> device address
        for r, rb in enumerate(allb):
            row = []
            for i, (hb, off) in enumerate(rb):
                if r == self.rank:
                    row.append(tensors[i].data_ptr())
                    continue
                h = (ctypes.c_ubyte * hsz).from_buffer_copy(hb)
                p = ctypes.c_void_p()
                _lib.check(lib.rm_ipc_open_handle(ctypes.addressof(h), ctypes.byref(p)),
                           "rm_ipc_open_handle")
                self._opened.append(p.value)
                row.append(p.value + off)
            self.bases.append(row)

    def close(self):
        lib = _lib.load()
        for p in self._opened:
            lib.rm_ipc_close_handle(ctypes.c_void_p(p))
        self._opened = []


def _peer_table(handle, device) -> torch.Tensor:
    """Device uint64[world]: every rank's address of a symmetric buffer."""
    off = int(getattr(handle, "offset", 0) or 0)
    peers = np.array([int(p) + off for p in handle.buffer_ptrs], dtype=np.uint64)
    return torch.from_numpy(peers.view(np.int64)).to(device)


def _use_multicast(handle) -> bool:
    """NVSwitch multicast when the handle has it, unless RINGMIX_SYM_P2P=1 forces the
    peer-table (unicast P2P) form (used by the multi-GPU checks to run both)."""
    return bool(handle.multicast_ptr) and os.environ.get("RINGMIX_SYM_P2P", "0") != "1"


def _sym_addresses(handle, device) -> tuple[int, torch.Tensor | None]:
    """(multicast address, None) when NVSwitch multicast is used, else (0, peer table)."""
    if _use_multicast(handle):
        return int(handle.multicast_ptr) + int(getattr(handle, "offset", 0) or 0), None
    return 0, _peer_table(handle, device)


class StepSync:
    """In-kernel ordering of consecutive learner-sharded steps (rm_step_sync): a flag in
    symmetric memory counts finished steps of all ranks; each step kernel waits for the
    previous step of every rank and bumps every rank's flag when it is done — through
    NVSwitch multicast, or one unicast P2P atomic per rank (peer table) where multicast
    is unavailable.  Replaces a host-issued barrier collective between steps.

    Epochs advance only when a launch succeeded (`begin` / `commit`), so a rejected
    launch does not leave every later wait target unreachable."""

    def __init__(self, group, device):
        import torch.distributed._symmetric_memory as symm_mem

        self.group = group if group is not None else dist.group.WORLD
        self.device = device
        self.world = dist.get_world_size(self.group)
        self.flag = symm_mem.empty(4, dtype=torch.int32, device=device)
        self.flag.zero_()
        self.handle = symm_mem.rendezvous(self.flag, self.group.group_name)
        self.mc, self.peers = _sym_addresses(self.handle, device)
        self.counter = torch.zeros(4, dtype=torch.int32, device=device)
        self.epoch = 0
        torch.cuda.synchronize(device)
        dist.barrier(group=self.group)   # every rank's flag is zero before any bump

    @property
    def multicast(self) -> bool:
        return bool(self.mc)

    def begin(self) -> "_lib.StepSyncArgs":
        """Arguments of the next step (epoch + 1); call `commit` once it launched."""
        return self._args(self.epoch + 1)

    def commit(self) -> None:
        self.epoch += 1

    def _args(self, epoch: int) -> "_lib.StepSyncArgs":
        return _lib.StepSyncArgs(self.flag.data_ptr(), self.mc or None, self.counter.data_ptr(),
                                 epoch, self.world,
                                 None if self.peers is None else self.peers.data_ptr())

    def wait_all(self) -> None:
        """Stream-ordered: later work on the current stream starts once every rank
        finished the latest step (rm_step_sync_wait)."""
        _lib.check(_lib.load().rm_step_sync_wait(ctypes.byref(self._args(self.epoch)),
                                                 _lib.stream_ptr()), "rm_step_sync_wait")

    def publish(self) -> None:
        """Collective, stream-ordered: every rank's next step waits for the writes this
        rank issued on the current stream before the call (rm_step_sync_publish)."""
        _lib.check(_lib.load().rm_step_sync_publish(ctypes.byref(self.begin()),
                                                    _lib.stream_ptr()), "rm_step_sync_publish")
        self.commit()


def _make_step_sync(group, device, enabled):
    if not enabled or os.environ.get("RINGMIX_STEP_SYNC", "1") == "0":
        return None
    try:
        return StepSync(group, device)
    except Exception:
        return None


class LearnerShardedRing:
    """RAD / fixed-ring step with learners sharded over the ranks of `group`.

    Holds the two W buffers (learner-major, this rank's Lg rows) and the
    IPC row-pointer tables; `step(...)` runs plan -> fused mix -> step barrier.
    """

    def __init__(self, L: int, d: int, dtype=torch.float32, group=None, device=None,
                 step_sync: bool = True, fixed_ring: bool = False):
        """fixed_ring: every step uses the fixed ring (AD-PSGD / D-PSGD), whose contiguous
        shards pull at most their 2 boundary rows — the kernel's stages then need no room for
        more (rm_set_shard_remote_rows), which lets them hold 1 KB row segments."""
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed must be initialised")
        self.fixed_ring = fixed_ring
        _lib.require_cuda()
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.L, self.d, self.dtype = L, d, dtype
        self.layout = ShardLayout(L, self.world)
        self.row0, row1 = self.layout.rows(self.rank)
        self.Lg = row1 - self.row0
        if self.Lg < 1:
            raise ValueError(f"need at least one learner per rank (L={L}, world={self.world})")
        self.device = torch.device(device if device is not None else
                                   f"cuda:{torch.cuda.current_device()}")
        self.W = [mixing.empty_learner_major(self.Lg, d, dtype, self.device) for _ in range(2)]
        self.ld = self.W[0].stride(0)
        self.peers = PeerMappedBuffers(self.W, group)
        esz = torch.empty((), dtype=dtype).element_size()
        self.row_ptrs = []
        for parity in range(2):
            ptrs = np.empty(L, dtype=np.uint64)
            for r, (b, e) in enumerate(self.layout.bounds):
                base = self.peers.bases[r][parity]
                for i in range(e - b):
                    ptrs[b + i] = base + i * self.ld * esz
            self.row_ptrs.append(torch.from_numpy(ptrs.view(np.int64)).to(self.device))
        self.plan = torch.empty(_lib.load().rm_shard_plan_ints(self.Lg), dtype=torch.int32,
                                device=self.device)
        self._token = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.cur = 0
        self._fn = getattr(_lib.load(), f"rm_ring_mix_sgd_sharded_{mixing._suffix(self.W[0])}")
        # consecutive steps ordered inside the kernel when multicast is available
        self.sync = _make_step_sync(group, self.device, step_sync)

    @property
    def weights(self) -> torch.Tensor:
        """This rank's learners, learner-major (Lg, d)."""
        return self.W[self.cur]

    def barrier(self):
        """Stream-ordered step barrier: every rank's previous kernels are complete
        (and their W' rows readable by peers) when this returns on the stream.  A
        no-op when the step kernels order themselves (StepSync)."""
        if self.sync is None:
            dist.all_reduce(self._token, group=self.group)

    def settle(self):
        """Order later work on the current stream after every rank's last step (a reader
        that must see the whole step of every rank; the local outputs alone need no
        wait)."""
        if self.sync is not None:
            self.sync.wait_all()

    def publish(self):
        """Collective: call on every rank after writing this rank's current rows from
        outside the step (initial weights, restore); the next step of every rank — whose
        pulls read these rows — is ordered after the writes.  In-kernel ordering: a
        stream-ordered flag bump (rm_step_sync_publish); otherwise a device sync and a
        barrier."""
        _publish(self)

    def step(self, left: torch.Tensor, right: torch.Tensor, G: torch.Tensor | None, lr: float,
             absmax: torch.Tensor | None = None, barrier: bool = True) -> torch.Tensor:
        """One step: W[cur] -> W[1-cur].  left/right: device int32[L] global tables."""
        lib = _lib.load()
        s = _lib.stream_ptr()
        _lib.check(lib.rm_shard_plan(left.data_ptr(), right.data_ptr(), self.L, self.row0,
                                     self.Lg, self.plan.data_ptr(), s), "rm_shard_plan")
        src, dst = self.W[self.cur], self.W[1 - self.cur]
        if G is not None:
            mixing._same(src, G, "G")
        ldg = G.stride(0) if G is not None else self.ld
        args = None if self.sync is None else self.sync.begin()
        if self.fixed_ring:
            _lib.check(lib.rm_set_shard_remote_rows(2), "rm_set_shard_remote_rows")
        try:
            _lib.check(self._fn(self.row_ptrs[self.cur].data_ptr(), src.data_ptr(),
                                _lib.ptr(G), dst.data_ptr(), self.L, self.row0, self.Lg,
                                self.d, self.ld, ldg, dst.stride(0), self.plan.data_ptr(),
                                float(lr), _lib.ptr(absmax), s,
                                None if args is None else ctypes.byref(args)),
                       "rm_ring_mix_sgd_sharded")
        finally:
            if self.fixed_ring:
                lib.rm_set_shard_remote_rows(0)
        if self.sync is not None:
            self.sync.commit()
        self.cur = 1 - self.cur
        if barrier:
            self.barrier()
        return dst

    def close(self):
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        self.peers.close()


def _publish(obj) -> None:
    if obj.sync is not None:
        obj.sync.publish()
    else:
        torch.cuda.synchronize(obj.device)
        dist.barrier(group=obj.group)


def _slot_table(layout: "ShardLayout", bases: list[int], ld: int, esz: int,
                device) -> torch.Tensor:
    """Device uint64[L]: address of slot/row x on its owning rank."""
    ptrs = np.empty(layout.L, dtype=np.uint64)
    for r, (b, e) in enumerate(layout.bounds):
        for i in range(e - b):
            ptrs[b + i] = bases[r] + i * ld * esz
    return torch.from_numpy(ptrs.view(np.int64)).to(device)


class LearnerShardedRingPos:
    """RAD with learners stored in ring-POSITION order (SURVEY §8(e) "push").

    Rank g owns Lg slots; at step k they hold a contiguous arc of ring positions of p_k
    (slot i: position ``slot_positions()[i]``, learner ``slot_learners(inv_k)[i]``).  The
    mix reads only the two boundary slots from the neighbouring ranks, and each output is
    stored straight into the learner's slot for step k+1 on whichever rank owns it — so a
    step moves ~Lg (n-1)/n + 2 rows over NVLink per rank instead of the ~2 Lg (n-1)/n the
    learner-ordered pull needs.  Where the arcs of step k+1 start and which rank gets which
    arc is free (the mix only sees neighbour relations): with equal shards every step picks
    the rotation and arc -> rank assignment that keeps the most learners on the rank that
    computes them (``rm_pos_placement``, deterministic on every rank; ~15 % fewer
    relabelling stores than slot x = position x).  Bit-identical to the single-GPU step.
    """

    def __init__(self, L: int, d: int, dtype=torch.float32, group=None, device=None,
                 step_sync: bool = True, placement: str | None = None):
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed must be initialised")
        _lib.require_cuda()
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.L, self.d, self.dtype = L, d, dtype
        self.layout = ShardLayout(L, self.world)
        self.g0, g1 = self.layout.rows(self.rank)
        self.Lg = g1 - self.g0
        if self.Lg < 1 or L < 4:
            raise ValueError(f"need L >= 4 and a position per rank (L={L}, world={self.world})")
        self.device = torch.device(device if device is not None else
                                   f"cuda:{torch.cuda.current_device()}")
        self.W = [mixing.empty_learner_major(self.Lg, d, dtype, self.device) for _ in range(2)]
        self.ld = self.W[0].stride(0)
        self.peers = PeerMappedBuffers(self.W, group)
        esz = torch.empty((), dtype=dtype).element_size()
        self.slots = [_slot_table(self.layout, [self.peers.bases[r][p] for r in range(self.world)],
                                  self.ld, esz, self.device) for p in range(2)]
        lib = _lib.load()
        self.plan = torch.empty(lib.rm_shard_plan_ints(self.Lg), dtype=torch.int32,
                                device=self.device)
        self.dest = torch.empty(self.Lg, dtype=torch.int64, device=self.device)
        self._token = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.cur = 0
        self._fn = getattr(lib, f"rm_ring_mix_sgd_pos_{mixing._suffix(self.W[0])}")
        self.sync = _make_step_sync(group, self.device, step_sync)
        # arc placement (rotation + arc -> rank per step, chosen to keep learners local):
        # needs equal shards; RINGMIX_POS_PLACEMENT=fixed keeps slot x = position x
        if placement is None:
            placement = os.environ.get("RINGMIX_POS_PLACEMENT", "rotate")
        self.placed = (placement == "rotate" and self.world > 1 and L % self.world == 0
                       and self.world <= 8 and L <= 1024)
        ident = torch.arange(L, dtype=torch.int32, device=self.device)
        # [pos_of_slot, slot_of_pos] for the current and the next step
        self.place = [[ident.clone(), ident.clone()], [ident.clone(), ident.clone()]]
        self.pc = 0
        self.moved = torch.zeros(self.world, dtype=torch.int32, device=self.device)
        self.moved_log: list[torch.Tensor] = []

    @property
    def slots_local(self) -> torch.Tensor:
        """This rank's slots (learner-major rows, ring-position order of the current step).
        Every rank writes into them, so with in-kernel step ordering the current stream
        first waits for every rank's last step (`settle`)."""
        self.settle()
        return self.W[self.cur]

    def settle(self):
        """Order later work on the current stream after every rank's last step (every rank
        writes into this rank's slots): readers of the slots, and writers before they
        overwrite them."""
        if self.sync is not None:   # (without it every step ends in a collective barrier)
            self.sync.wait_all()

    def publish(self):
        """Collective: after writing this rank's current slots from outside the step
        (`settle` first), order every rank's next step — which reads the boundary slots —
        after the writes."""
        _publish(self)

    def barrier(self):
        """Step barrier on the stream (a no-op when the kernels order themselves)."""
        if self.sync is None:
            dist.all_reduce(self._token, group=self.group)

    def step(self, inv_k: torch.Tensor, perm_next: torch.Tensor, G: torch.Tensor | None,
             lr: float, absmax: torch.Tensor | None = None, barrier: bool = True):
        """inv_k: device int32[L] (learner at each position, step k); perm_next:
        device int32[L] (position of each learner at step k+1); G: this rank's
        gradients in slot order (Lg, d)."""
        lib = _lib.load()
        s = _lib.stream_ptr()
        if self.placed:
            cur, nxt = self.place[self.pc], self.place[1 - self.pc]
            _lib.check(lib.rm_pos_placement(inv_k.data_ptr(), perm_next.data_ptr(),
                                            cur[1].data_ptr(), self.L, self.world,
                                            nxt[0].data_ptr(), nxt[1].data_ptr(),
                                            self.moved.data_ptr(), s), "rm_pos_placement")
            _lib.check(lib.rm_pos_plan_placed(inv_k.data_ptr(), perm_next.data_ptr(),
                                              cur[0].data_ptr(), cur[1].data_ptr(),
                                              nxt[1].data_ptr(), self.L, self.g0, self.Lg,
                                              self.slots[1 - self.cur].data_ptr(),
                                              self.plan.data_ptr(), self.dest.data_ptr(), s),
                       "rm_pos_plan_placed")
        else:
            _lib.check(lib.rm_pos_plan(inv_k.data_ptr(), perm_next.data_ptr(), self.L, self.g0,
                                       self.Lg, self.slots[1 - self.cur].data_ptr(),
                                       self.plan.data_ptr(), self.dest.data_ptr(), s),
                       "rm_pos_plan")
        src = self.W[self.cur]
        if G is not None:
            mixing._same(src, G, "G")
        args = None if self.sync is None else self.sync.begin()
        _lib.check(self._fn(self.slots[self.cur].data_ptr(), src.data_ptr(), _lib.ptr(G), self.L,
                            self.g0, self.Lg, self.d, self.ld,
                            G.stride(0) if G is not None else self.ld, self.plan.data_ptr(),
                            self.dest.data_ptr(), float(lr), _lib.ptr(absmax), s,
                            None if args is None else ctypes.byref(args)),
                   "rm_ring_mix_sgd_pos")
        if self.sync is not None:
            self.sync.commit()
        self.cur = 1 - self.cur
        if self.placed:
            self.pc = 1 - self.pc
            if self.log_moves:
                self.moved_log.append(self.moved.clone())
        if barrier:
            self.barrier()

    log_moves = False

    def slot_positions(self) -> torch.Tensor:
        """Ring positions held by this rank's slots at the current step (device int32[Lg]):
        slot i holds the learner inv_k[slot_positions()[i]]."""
        return self.place[self.pc][0][self.g0:self.g0 + self.Lg]

    def slot_learners(self, inv_k: torch.Tensor) -> torch.Tensor:
        """Learner ids in this rank's slots for the current step, given that step's inv_k
        (e.g. to produce their gradients in slot order)."""
        return inv_k[self.slot_positions().long()]

    def close(self):
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        self.peers.close()


class LearnerShardedD1DNVLS:
    """D1D step with learners sharded, the cross-GPU sum done by our own kernel in the
    NVSwitch: every rank writes its fp64 column partial sums into a symmetric buffer;
    for its 1/N column shard a rank sums all ranks' partials in the switch
    (``multimem.ld_reduce``) and broadcasts the totals into every rank's copy
    (``multimem.st``); then each rank applies mean - lr*G to its learners.  No NCCL
    kernels; the cross-rank barriers are symmetric-memory signal pads (stream-ordered).

    The columns are cut into chunks (``chunk_cols``; None = one chunk) and pipelined
    over two streams, so the in-switch reduction of chunk c (side stream) overlaps
    the partial sums of chunk c+1 and the apply of chunk c-1 (compute stream) — the
    D1D global average overlapped with the local update (north-star (c))."""

    MAX_CHUNKS = 16   # barrier channels per handle: torch allows 32

    def __init__(self, L: int, d: int, Lg: int, device, group=None,
                 chunk_cols: int | None = 1 << 22):
        import torch.distributed._symmetric_memory as symm_mem

        self.L, self.d, self.Lg = L, d, Lg
        self.device = torch.device(device)
        self.group = group if group is not None else dist.group.WORLD
        gname = self.group.group_name
        self.rank = dist.get_rank(self.group)
        self.world = dist.get_world_size(self.group)
        self.P = symm_mem.empty(d, dtype=torch.float64, device=self.device)
        self.M = symm_mem.empty(d, dtype=torch.float64, device=self.device)
        self.hP = symm_mem.rendezvous(self.P, gname)
        self.hM = symm_mem.rendezvous(self.M, gname)
        if not self.hP.multicast_ptr or not self.hM.multicast_ptr:
            raise RuntimeError("NVSwitch multicast (NVLS) is not available on this system")
        # chunk boundaries on multiples of 32*world columns; inside a chunk every rank
        # reduces a 1/N slice with 32-column (256 B) aligned boundaries
        quantum = 32 * self.world
        want = d if chunk_cols is None else max(quantum, chunk_cols)
        want = max(want, -(-d // self.MAX_CHUNKS))
        step = -(-want // quantum) * quantum
        self.chunks = [(c, min(c + step, d)) for c in range(0, d, step)] or [(0, 0)]
        self.shards = []
        for b, e in self.chunks:
            sl = -(-(e - b) // self.world)
            sl = -(-sl // 32) * 32
            c0 = min(e, b + self.rank * sl)
            self.shards.append((c0, min(e, c0 + sl)))
        # kept for callers that read the single-chunk shard
        self.c0, self.c1 = self.shards[0]
        self.comm = torch.cuda.Stream(device=self.device)
        # co-residency of the pipelined kernels: (local partial-sum/apply, in-switch)
        # (partial sum, apply, in-switch reduce); apply needs 75 registers per thread
        env = os.environ.get("RINGMIX_D1D_CTAS", "4,2,2").split(",")
        self.ctas_per_sm = tuple(int(x) for x in env)
        # numpy-order partial sums (bit-identical to the one-GPU mean); local rows then hold
        # d1d_learners(L, world, rank, chains).  Up to 2 ranks the in-switch sum is exact;
        # above, the reduction runs over peer tables in the tree order (rm_p2p_mean_f64) —
        # at 4 ranks by default, at 8 on request (same rule as LearnerShardedD1DFused)
        want = os.environ.get("RINGMIX_D1D_NUMPY_ORDER", "auto")
        self.chains = d1d_numpy_chains(L, self.world) if (
            self.world <= 4 or want == "1") else 0
        self.p2p = bool(self.chains) and self.world > 2
        if self.p2p:
            self.tP, self.tM = _peer_table(self.hP, self.device), _peer_table(self.hM, self.device)

    def _launch_partial(self, W: torch.Tensor, i: int, stream) -> torch.cuda.Event:
        """Partial sums of chunk i on `stream`, then (comm stream) the in-switch mean of this
        rank's slice of it; returns the event after which every rank's means of chunk i are
        in M."""
        lib = _lib.load()
        b, e = self.chunks[i]
        esz = W.element_size()
        psum = getattr(lib, f"rm_partial_sum_{mixing._suffix(W)}")
        with _NumpyOrder(self.chains if W.element_size() >= 4 else 0):
            _lib.check(psum(W.data_ptr() + b * esz, self.Lg, e - b, W.stride(0),
                            self.P.data_ptr() + b * 8, stream.cuda_stream), "rm_partial_sum")
        ev = torch.cuda.Event()
        ev.record(stream)
        self.comm.wait_event(ev)
        c0, c1 = self.shards[i]
        with torch.cuda.stream(self.comm):
            self.hP.barrier(channel=i)          # every rank's partials of chunk i
            if self.p2p:
                with _NumpyOrder(self.chains):  # tree order over the ranks
                    _lib.check(lib.rm_p2p_mean_f64(self.tP.data_ptr(), self.tM.data_ptr(),
                                                   self.world, c0, c1, self.L,
                                                   self.comm.cuda_stream), "rm_p2p_mean_f64")
            else:
                _lib.check(lib.rm_nvls_mean_f64(self.hP.multicast_ptr, self.hM.multicast_ptr,
                                                c0, c1, self.L, self.comm.cuda_stream),
                           "rm_nvls_mean_f64")
            self.hM.barrier(channel=i)          # every rank's means of chunk i
            done = torch.cuda.Event()
            done.record(self.comm)
        return done

    def _launch_apply(self, W, G, lr, out, absmax, i: int, ready, stream) -> None:
        lib = _lib.load()
        apply = getattr(lib, f"rm_apply_mean_sgd_{mixing._suffix(W)}")
        b, e = self.chunks[i]
        esz = W.element_size()
        stream.wait_event(ready)
        # M holds the means already (L = 1: no per-learner division)
        gp = None if G is None else G.data_ptr() + b * esz
        _lib.check(apply(self.M.data_ptr() + b * 8, gp, out.data_ptr() + b * esz, self.Lg,
                         1, e - b, G.stride(0) if G is not None else 0, out.stride(0),
                         float(lr), _lib.ptr(absmax), stream.cuda_stream),
                   "rm_apply_mean_sgd")

    def mean_async(self, W: torch.Tensor, stream) -> list[torch.cuda.Event]:
        """The global column means of W (every rank's learners) into M, launched on
        `stream` (partial sums) and the comm stream (in-switch reduction); returns one
        event per chunk.  Pair with ``apply``."""
        return [self._launch_partial(W, i, stream) for i in range(len(self.chunks))]

    def apply(self, W: torch.Tensor, G: torch.Tensor | None, lr: float, out: torch.Tensor,
              ready: list[torch.cuda.Event], absmax: torch.Tensor | None = None) -> torch.Tensor:
        """out = M - lr * G on the current stream, chunk by chunk after `ready`."""
        compute = torch.cuda.current_stream(self.device)
        for i in range(len(self.chunks)):
            self._launch_apply(W, G, lr, out, absmax, i, ready[i], compute)
        return out

    def step(self, W: torch.Tensor, G: torch.Tensor | None, lr: float, out: torch.Tensor,
             absmax: torch.Tensor | None = None) -> torch.Tensor:
        lib = _lib.load()
        compute = torch.cuda.current_stream(self.device)
        ready: list[torch.cuda.Event] = []

        def launch_partial(i):
            ready.append(self._launch_partial(W, i, compute))

        def launch_apply(i):
            self._launch_apply(W, G, lr, out, absmax, i, ready[i], compute)

        n = len(self.chunks)
        if n > 1:
            _lib.check(lib.rm_set_d1d_ctas_per_sm(*self.ctas_per_sm), "rm_set_d1d_ctas_per_sm")
        try:
            launch_partial(0)
            for i in range(n):
                if i + 1 < n:
                    launch_partial(i + 1)
                launch_apply(i)
        finally:
            if n > 1:
                lib.rm_set_d1d_ctas_per_sm(0, 0, 0)
        return out


class LearnerShardedD1DFused:
    """D1D step with learners sharded, everything in ONE kernel launch per rank
    (``rm_d1d_fused_nvls_*``): the CTAs split into partial-sum, in-switch-reduce and
    apply roles that walk the column chunks in order and hand each chunk on — within
    the GPU through counters, across GPUs through flags bumped on every rank with
    ``multimem.red``.  The reduction of chunk c in the NVSwitch overlaps the partial
    sums of later chunks and the apply of earlier ones without any host-side stream
    choreography; the arithmetic is that of LearnerShardedD1DNVLS (same bits)."""

    MAX_CHUNKS = 64

    def __init__(self, L: int, d: int, Lg: int, device, group=None,
                 chunk_cols: int = 1 << 21, split: tuple[int, int] | None = None):
        import torch.distributed._symmetric_memory as symm_mem

        self.L, self.d, self.Lg = L, d, Lg
        self.device = torch.device(device)
        self.group = group if group is not None else dist.group.WORLD
        gname = self.group.group_name
        self.rank = dist.get_rank(self.group)
        self.world = dist.get_world_size(self.group)
        self.P = symm_mem.empty(max(d, 1), dtype=torch.float64, device=self.device)
        self.M = symm_mem.empty(max(d, 1), dtype=torch.float64, device=self.device)
        self.F = symm_mem.empty(2 * self.MAX_CHUNKS, dtype=torch.int32, device=self.device)
        self.F.zero_()
        self.hP = symm_mem.rendezvous(self.P, gname)
        self.hM = symm_mem.rendezvous(self.M, gname)
        self.hF = symm_mem.rendezvous(self.F, gname)
        # NVSwitch multicast when available (in-switch reduction), else peer tables
        # (unicast NVLink loads / stores, rm_d1d_fused_p2p_*)
        handles = (self.hP, self.hM, self.hF)
        self.multicast = all(_use_multicast(h) for h in handles)
        # numpy order (the one-GPU step's bits): free with the in-switch sum up to 2 ranks;
        # above that the tree runs over peer tables — the default at 4 ranks (measured 1,001
        # vs 1,032 G/s for the in-switch sum at C4, profiles/r3_p2psplit/), on request at 8
        # (RINGMIX_D1D_NUMPY_ORDER=1; not measured on 8 GPUs)
        self.chains = d1d_numpy_chains(L, self.world, multicast_reduce=self.multicast)
        want = os.environ.get("RINGMIX_D1D_NUMPY_ORDER", "auto")
        if (not self.chains and self.multicast and self.world > 2 and want != "0"
                and (self.world <= 4 or want == "1")):
            self.chains = d1d_numpy_chains(L, self.world)
            if self.chains:
                self.multicast = False
        self._sym = [_sym_addresses(h, self.device) if self.multicast
                     else (0, _peer_table(h, self.device)) for h in handles]
        self.counters = torch.zeros(2 * self.MAX_CHUNKS, dtype=torch.int32, device=self.device)
        quantum = 32 * self.world
        chunk_cols = int(os.environ.get("RINGMIX_D1D_FUSED_CHUNK", chunk_cols))
        chunk = max(chunk_cols, -(-d // self.MAX_CHUNKS), quantum)
        self.chunk = -(-chunk // quantum) * quantum
        if split is None:
            # CTA shares (partial sums, reduction; the rest apply): the in-switch reduction
            # needs few CTAs, the peer-table reduction (world loads + world stores per
            # column) many — 20 / 40 measured 1,001 vs 433 G/s for 30 / 10 at n = 4
            dflt = "30,10" if self.multicast else "20,40"
            env = os.environ.get("RINGMIX_D1D_FUSED_SPLIT", dflt).split(",")
            split = (int(env[0]), int(env[1]))
        self.split = split
        self.epoch = 0
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)     # every rank's flags are zero before any bump

    @property
    def chunks(self) -> list[tuple[int, int]]:
        return [(b, min(b + self.chunk, self.d)) for b in range(0, self.d, self.chunk)]

    def step(self, W: torch.Tensor, G: torch.Tensor | None, lr: float, out: torch.Tensor,
             absmax: torch.Tensor | None = None) -> torch.Tensor:
        lib = _lib.load()
        sfx = mixing._suffix(W)
        epoch = self.epoch + 1       # committed only once the launch succeeded
        ldg = G.stride(0) if G is not None else 0
        with _NumpyOrder(self.chains if W.element_size() >= 4 else 0):
            self._launch(lib, sfx, W, G, ldg, lr, out, absmax, epoch)
        self.epoch = epoch
        return out

    def _launch(self, lib, sfx, W, G, ldg, lr, out, absmax, epoch):
        if self.multicast:
            (pmc, _), (mmc, _), (fmc, _) = self._sym
            _lib.check(getattr(lib, f"rm_d1d_fused_nvls_{sfx}")(
                W.data_ptr(), _lib.ptr(G), out.data_ptr(), self.Lg, self.L, self.d, W.stride(0),
                ldg, out.stride(0), float(lr), _lib.ptr(absmax), self.P.data_ptr(), pmc,
                self.M.data_ptr(), mmc, self.F.data_ptr(), fmc, self.counters.data_ptr(),
                self.rank, self.world, self.chunk, self.MAX_CHUNKS, epoch, self.split[0],
                self.split[1], _lib.stream_ptr()), "rm_d1d_fused_nvls")
        else:
            r = _lib.D1DRank(W.data_ptr(), _lib.ptr(G), out.data_ptr(), _lib.ptr(absmax),
                             self.P.data_ptr(), self.M.data_ptr(), self.F.data_ptr(),
                             self.counters.data_ptr(), self.Lg, self.rank)
            (_, pt), (_, mt), (_, ft) = self._sym
            _lib.check(getattr(lib, f"rm_d1d_fused_p2p_{sfx}")(
                ctypes.byref(r), 1, self.L, self.d, W.stride(0), ldg, out.stride(0), float(lr),
                pt.data_ptr(), mt.data_ptr(), ft.data_ptr(), self.world, self.chunk,
                self.MAX_CHUNKS, epoch, self.split[0], self.split[1], _lib.stream_ptr()),
                "rm_d1d_fused_p2p")


class LearnerShardedD1D:
    """D1D step with learners sharded: W' = sum_all(W)/L - lr*G, the global sum by an
    NCCL all-reduce of fp64 column sums, pipelined in column chunks so the
    all-reduce of chunk c overlaps the local kernels of chunks c+1 / c-1."""

    def __init__(self, L: int, d: int, Lg: int, device, chunk_cols: int = 1 << 22, group=None):
        self.L, self.d, self.Lg, self.group = L, d, Lg, group
        self.device = torch.device(device)
        # chunk boundaries on 32-column (128 B) multiples keep every row 16 B aligned
        step = max(32, (chunk_cols // 32) * 32)
        self.chunks = [(b, min(b + step, d)) for b in range(0, d, step)]
        self.S = torch.empty(d, dtype=torch.float64, device=self.device)
        self.comm = torch.cuda.Stream(device=self.device)
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.chains = d1d_numpy_chains(L, world, multicast_reduce=True)
        # co-residency of the pipelined kernels: (local partial-sum/apply, in-switch)
        # (partial sum, apply, in-switch reduce); apply needs 75 registers per thread
        env = os.environ.get("RINGMIX_D1D_CTAS", "4,2,2").split(",")
        self.ctas_per_sm = tuple(int(x) for x in env)

    def step(self, W: torch.Tensor, G: torch.Tensor | None, lr: float, out: torch.Tensor,
             absmax: torch.Tensor | None = None) -> torch.Tensor:
        lib = _lib.load()
        sfx = mixing._suffix(W)
        psum = getattr(lib, f"rm_partial_sum_{sfx}")
        apply = getattr(lib, f"rm_apply_mean_sgd_{sfx}")
        compute = torch.cuda.current_stream(self.device)
        esz = W.element_size()
        ready = []

        def launch_partial(i):
            b, e = self.chunks[i]
            with _NumpyOrder(self.chains if W.element_size() >= 4 else 0):
                _lib.check(psum(W.data_ptr() + b * esz, self.Lg, e - b, W.stride(0),
                                self.S.data_ptr() + b * 8, compute.cuda_stream),
                           "rm_partial_sum")
            ev = torch.cuda.Event()
            ev.record(compute)
            self.comm.wait_event(ev)
            with torch.cuda.stream(self.comm):
                dist.all_reduce(self.S[b:e], group=self.group)
                done = torch.cuda.Event()
                done.record(self.comm)
            ready.append(done)

        def launch_apply(i):
            b, e = self.chunks[i]
            compute.wait_event(ready[i])
            gp = 0 if G is None else G.data_ptr() + b * esz
            _lib.check(apply(self.S.data_ptr() + b * 8, gp or None, out.data_ptr() + b * esz,
                             self.Lg, self.L, e - b, G.stride(0) if G is not None else 0,
                             out.stride(0), float(lr), _lib.ptr(absmax), compute.cuda_stream),
                       "rm_apply_mean_sgd")

        n = len(self.chunks)
        for i in range(n):
            launch_partial(i)
            if i >= 1:
                launch_apply(i - 1)
        launch_apply(n - 1)
        return out


class ShardedD1DTrainer:
    """One D1D training step of a learner-sharded run with a device oracle
    (simulation.py:304-312 with gradient_matrix :226-238):
        W_{k+1}[local] = mean_all(W_k) - lr * G(W_{k-1}[local])
    The paper's D1D concurrency: the global average of W_k does not
    depend on the gradient, so with ``overlap`` it runs — partial sums on a side stream,
    the in-switch reduction on the NVLS comm stream (LearnerShardedD1DNVLS.mean_async) —
    concurrently with the oracle's gradient of W_{k-1} on the compute stream (the average's
    kernels capped at ``ctas`` CTAs per SM so they run beside the generator instead of
    displacing it), and the generator's final pass writes M - lr G itself (``fuse_grad``,
    rm_quadratic_mean_step_shard_*; else G goes to HBM and one apply pass follows).  Default:
    overlapped and fused, measured 8.28 vs 8.93 ms serial at C4 on 2 GPUs.
    Without ``overlap`` the gradient runs first, then the single-kernel fused D1D step
    (LearnerShardedD1DFused).  All modes give the same bits.
    learner0: this rank's first learner (its rows draw the gradient streams
    learner0 + l) — with the numpy-order D1D sharding (``chains`` > 0, the default where it
    is exact) local row i is learner d1d_learners(L, world, rank, chains)[i] instead, and
    the generator draws those learners' streams (rm_set_shard_streams)."""

    def __init__(self, L: int, d: int, Lg: int, learner0: int, device, oracle, group=None,
                 overlap: bool | None = None, ctas: tuple[int, int, int] | None = None,
                 fuse_grad: bool | None = None):
        self.L, self.d, self.Lg, self.learner0 = L, d, Lg, learner0
        # overlap + fuse_grad: the generator's final pass writes W' = M - lr G itself
        # (rm_quadratic_mean_step_shard_*), so G never reaches HBM and no apply pass runs
        if fuse_grad is None:
            fuse_grad = os.environ.get("RINGMIX_D1D_TRAIN_FUSED", "1") == "1"
        self.fuse_grad = fuse_grad
        # CTAs per SM of the partial-sum / apply / in-switch kernels while they share the GPU
        # with the generator (0 = the kernels' defaults, which take whole SMs)
        if ctas is None:
            ctas = tuple(int(x) for x in
                         os.environ.get("RINGMIX_D1D_TRAIN_CTAS", "4,0,1").split(","))
        self.ctas = ctas
        self.device = torch.device(device)
        self.oracle = oracle
        if overlap is None:
            overlap = os.environ.get("RINGMIX_D1D_TRAIN_OVERLAP", "1") == "1"
        self.overlap = overlap
        split = overlap or fuse_grad   # the average as its own pipeline (mean_async)
        self.nvls = LearnerShardedD1DNVLS(L, d, Lg, device, group=group) if split else None
        self.fused = None if split else LearnerShardedD1DFused(L, d, Lg, device, group=group)
        self.chains = (self.nvls or self.fused).chains
        if self.chains:
            self.learner0 = dist.get_rank(group) * self.chains
        # high priority: the memory-bound partial sums take SM slots as the compute-bound
        # generator's CTAs retire instead of queueing behind all of them
        self.side = torch.cuda.Stream(device=self.device, priority=-1)
        self.G = None

    def step(self, W: torch.Tensor, W_prev: torch.Tensor, cfg, k: int, lr: float,
             out: torch.Tensor, absmax: torch.Tensor | None = None) -> torch.Tensor:
        main = torch.cuda.current_stream(self.device)
        if self.G is None or self.G.shape != W.shape or self.G.dtype != W.dtype:
            self.G = mixing.empty_learner_major(self.Lg, self.d, W.dtype, self.device)
        if self.fused is not None:
            with _ShardStreams(self.chains):
                G = self.oracle.device_gradients(W_prev, cfg, k, learner0=self.learner0,
                                                 out=self.G)
            return self.fused.step(W, G, lr, out, absmax=absmax)
        lib = _lib.load()
        if self.overlap:
            self.side.wait_stream(main)
            _lib.check(lib.rm_set_d1d_ctas_per_sm(*self.ctas), "rm_set_d1d_ctas_per_sm")
            try:
                ready = self.nvls.mean_async(W, self.side)
            finally:
                lib.rm_set_d1d_ctas_per_sm(0, 0, 0)
        else:   # the average first, then the gradient (fused or not)
            ready = self.nvls.mean_async(W, main)
        if self.fuse_grad and W.dtype in (torch.float32, torch.float64):
            self._fused_mean_step(W_prev, cfg, k, lr, out, ready[-1], absmax)
        else:
            with _ShardStreams(self.chains):
                G = self.oracle.device_gradients(W_prev, cfg, k, learner0=self.learner0,
                                                 out=self.G)
            self.nvls.apply(W, G, lr, out, ready, absmax=absmax)
        main.wait_stream(self.side)
        return out

    def _fused_mean_step(self, W_prev, cfg, k, lr, out, ready, absmax):
        """out = M - lr * G(W_prev) with the gradient fused into the final pass; the
        generator runs now, its mix waits for `ready` (every chunk's global means)."""
        with _ShardStreams(self.chains):
            self.oracle.device_mean_step(self.nvls.M, W_prev, lr, cfg, k, ready=ready,
                                         learner0=self.learner0, absmax=absmax, out=out)

    def close(self):
        pass

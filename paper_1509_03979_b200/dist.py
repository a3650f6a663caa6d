"""Multi-GPU plumbing for batched recovery.

Independent problems shard across ranks (one process per GPU) in contiguous
blocks; each rank recovers its block with cs_recover_batched and the only
collective is one all-gather of fixed-size result records (support, values,
report) — NCCL over NVLink on GPUs, gloo in the CPU tests.  No data-path
collective: the recovery itself never communicates.
"""
from __future__ import annotations

from typing import Tuple


def shard(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block (b0, count) of `total` problems owned by `rank`; the first
    total % world ranks get one extra problem."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    b0 = rank * base + min(rank, extra)
    return b0, base + (1 if rank < extra else 0)


def record_bytes(K: int, value_itemsize: int, report_bytes: int = 40) -> int:
    return K * 4 + K * value_itemsize + report_bytes


def pack_records(support, values, report):
    """[B, K] int32 support, [B, K] values, [B, 40] uint8 report -> [B, rec] uint8."""
    import torch
    B = support.shape[0]
    return torch.cat([support.contiguous().view(torch.uint8).reshape(B, -1),
                      values.contiguous().view(torch.uint8).reshape(B, -1),
                      report.contiguous().reshape(B, -1)], dim=1)


def unpack_records(rec, K: int, value_dtype):
    import torch
    B = rec.shape[0]
    vs = torch.empty((), dtype=value_dtype).element_size()
    supp = rec[:, :4 * K].contiguous().view(torch.int32).reshape(B, K)
    vals = rec[:, 4 * K:4 * K + vs * K].contiguous().view(value_dtype).reshape(B, K)
    rep = rec[:, 4 * K + vs * K:].contiguous()
    return supp, vals, rep


def gather_records(rec, world: int, total: int = 0, out=None, group=None):
    """All-gather every rank's [B_r, rec] block into [total, rec] in rank order (= problem
    order for `shard`).  Blocks may differ by one problem (total % world != 0): each rank's
    block is padded to ceil(total / world) records for the collective and the padding is
    dropped afterwards.  total = 0 means world * B_r (equal blocks)."""
    import torch
    import torch.distributed as dist
    B_r, R = rec.shape
    if total <= 0:
        total = world * B_r
    per = -(-total // world)
    if B_r != per:
        pad = torch.zeros((per, R), dtype=rec.dtype, device=rec.device)
        pad[:B_r] = rec
        rec = pad
    flat = rec.contiguous().reshape(-1)
    if out is None or out.numel() != world * flat.numel():
        out = torch.empty(world * flat.numel(), dtype=flat.dtype, device=flat.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, flat, group=group)
    else:  # gloo: list form
        parts = list(out.chunk(world))
        dist.all_gather(parts, flat, group=group)
        out = torch.cat(parts)
    full = out.reshape(world, per, R)
    if per * world == total:
        return full.reshape(total, R)
    keep = [shard(total, r, world)[1] for r in range(world)]
    return torch.cat([full[r, :keep[r]] for r in range(world)])


# ------------------------------------------------------------------------------------------
# Single signal over G GPUs: the four-step operator of one large signal
# with one all-to-all per pass.  The [L1][L2] intermediate of the four-step FFT (L = N/2 =
# L1 L2, include/cs.h cs_dist_*) is split by column tiles for the column passes (A, C) and by
# row pairs (rows i and L1 - i, which the DCT split pairs) for the row pass (B); between them
# every rank sends each other rank the part of its columns that lies in that rank's rows.

class DistPlan:
    """Ownership of the distributed four-step operator: rank r owns the column tiles
    tiles[r] (columns cols[r], L2 / world of them) and the row-pair items items[r] (rows
    rows[r]).  Requires world to divide the L2 / CT column tiles."""

    def __init__(self, N: int, world: int, L1: int, L2: int, CT: int):
        ntiles, nitems = L2 // CT, L1 // 2 + 1
        if world < 1 or ntiles % world:
            raise ValueError(f"world {world} must divide the {ntiles} column tiles")
        self.N, self.world, self.L1, self.L2, self.CT = N, world, L1, L2, CT
        self.tiles = [(r * ntiles // world, (r + 1) * ntiles // world) for r in range(world)]
        self.cols = [(t0 * CT, t1 * CT) for t0, t1 in self.tiles]
        self.items = []
        for r in range(world):
            b0, cnt = shard(nitems, r, world)
            self.items.append((b0, b0 + cnt))
        self.rows = [self._rows(i0, i1) for i0, i1 in self.items]
        self.seg_len = L2 // world          # complex elements per segment (one row x one column block)

    def _rows(self, i0, i1):
        out = []
        for it in range(i0, i1):
            out.append(it)
            if it != 0 and it != self.L1 // 2:
                out.append(self.L1 - it)
        return out

    def y_ranges(self, rank: int, row_offsets):
        """[start, end) of this rank's entries in yT: its rows [i0, i1) and their partners
        L1 - i (items 0 < i < L1 / 2), each a contiguous block of rows in the transposed order
        (row_offsets[k1] = where row k1's entries start, cs_dist_row_offsets)."""
        i0, i1 = self.items[rank]
        out = [(row_offsets[i0], row_offsets[i1])] if i1 > i0 else []
        lo, hi = max(i0, 1), min(i1, self.L1 // 2)
        if hi > lo:
            out.append((row_offsets[self.L1 - hi + 1], row_offsets[self.L1 - lo + 1]))
        return out

    def segments(self, rank: int, direction: int, pack: bool):
        """(rows, col0, counts per peer) of the segments `rank` packs (pack=True) or unpacks.
        direction 0: after pass A, columns -> row pairs; 1: after pass B, row pairs -> columns.
        Segments are ordered by peer, so counts[p] consecutive segments go to / come from p
        (none to / from the rank itself: that block never leaves its workspace)."""
        rows, col0, counts = [], [], []
        for p in range(self.world):
            if p == rank:
                # this rank's own rows x own columns are already in place in its workspace
                counts.append(0)
                continue
            if direction == 0:
                # pack at the column owner `rank` for row owner p; unpack at row owner `rank` from p
                rs, c = (self.rows[p], self.cols[rank][0]) if pack else (self.rows[rank], self.cols[p][0])
            else:
                # pack at the row owner `rank` for column owner p; unpack at column owner `rank` from p
                rs, c = (self.rows[rank], self.cols[p][0]) if pack else (self.rows[p], self.cols[rank][0])
            rows += rs
            col0 += [c] * len(rs)
            counts.append(len(rs))
        return rows, col0, counts


def dist_plan(N: int, world: int) -> DistPlan:
    import ctypes
    from . import load_library
    L1, L2, CT = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
    rc = load_library().cs_dist_geometry(N, ctypes.byref(L1), ctypes.byref(L2), ctypes.byref(CT))
    if rc:
        raise RuntimeError(f"cs_dist_geometry: {load_library().cs_last_error().decode()}")
    return DistPlan(N, world, L1.value, L2.value, CT.value)


# phase ids (include/cs.h CS_DP_*)
DP_A, DP_BF, DP_BA, DP_C, DP_P, DP_YT, DP_XS, DP_XG = range(8)


class DistOperator:
    """One rank's share of the distributed operator of one signal (instance 0 of `op`, a plain
    P.DCT.diag(sigma) with N > 16384, fp32).  Vectors live in the distributed layouts of
    include/cs.h: x as this rank's "xc" (nxc reals on its columns), y as an [M] "yT" buffer of
    which only this rank's rows (y_ranges) are meaningful."""

    def __init__(self, op, plan: DistPlan, rank: int, row_offsets=None):
        import ctypes
        import torch
        from . import load_library
        self.op, self.plan, self.rank = op, plan, rank
        self.lib = load_library()
        dev = torch.device("cuda", torch.cuda.current_device())
        self.ws = torch.empty(int(self.lib.cs_dist_ws_bytes(op.N, op.M)), dtype=torch.uint8, device=dev)
        self.seg = {}
        for d in (0, 1):
            for pk in (True, False):
                rows, col0, counts = plan.segments(rank, d, pk)
                self.seg[(d, pk)] = (torch.tensor(rows, dtype=torch.int32, device=dev),
                                     torch.tensor(col0, dtype=torch.int32, device=dev),
                                     [2 * c * plan.seg_len for c in counts])
        t0, t1 = plan.tiles[rank]
        self.nxc = 2 * plan.L1 * (t1 - t0) * plan.CT
        if row_offsets is None:
            off = (ctypes.c_int64 * (plan.L1 + 1))()
            self._call(self.lib.cs_dist_row_offsets(op.handle, off), "cs_dist_row_offsets")
            row_offsets = list(off)
        self.row_offsets = row_offsets
        self.y_ranges = plan.y_ranges(rank, row_offsets)

    def _call(self, rc, what):
        if rc:
            raise RuntimeError(f"{what}: {self.lib.cs_last_error().decode()}")

    def phase(self, ph: int, inp=None, out=None):
        import ctypes
        import torch
        P = ctypes.c_void_p
        t0, t1 = self.plan.tiles[self.rank]
        i0, i1 = self.plan.items[self.rank]
        st = P(torch.cuda.current_stream().cuda_stream)
        self._call(self.lib.cs_dist_phase(self.op.handle, ph, t0, t1, i0, i1,
                                          P(inp.data_ptr()) if inp is not None else None,
                                          P(out.data_ptr()) if out is not None else None,
                                          P(self.ws.data_ptr()), self.ws.numel(), st), "cs_dist_phase")
        return out

    def copy(self, direction: int, pack: bool, buf):
        import ctypes
        import torch
        P = ctypes.c_void_p
        rows, col0, _ = self.seg[(direction, pack)]
        st = P(torch.cuda.current_stream().cuda_stream)
        self._call(self.lib.cs_dist_copy(self.op.handle, P(self.ws.data_ptr()), P(rows.data_ptr()),
                                         P(col0.data_ptr()), rows.numel(), self.plan.seg_len,
                                         P(buf.data_ptr()), 1 if pack else 0, st), "cs_dist_copy")

    def send_buffer(self, direction: int):
        import torch
        n = sum(self.seg[(direction, True)][2])
        buf = torch.empty(n, dtype=torch.float32, device=self.ws.device)
        self.copy(direction, True, buf)
        return buf, self.seg[(direction, True)][2], self.seg[(direction, False)][2]

    # layout changes (no arithmetic; entering / leaving the distributed layouts)
    def scatter_x(self, x):
        import torch
        return self.phase(DP_XS, inp=x, out=torch.empty(self.nxc, dtype=torch.float32, device=x.device))

    def scatter_y(self, y):
        import torch
        return self.phase(DP_YT, inp=y, out=torch.empty(self.op.M, dtype=torch.float32, device=y.device))

    def own_y(self, yT):
        """This rank's entries of yT, its two row blocks concatenated."""
        import torch
        return torch.cat([yT[a:b] for a, b in self.y_ranges])


def dist_apply(ranks, xcs, exchange):
    """y = A x for one signal: `ranks` = the DistOperator(s) this process plays (one under
    torchrun, several in the single-process emulation), xcs their x in the xc layout;
    exchange(sends) -> recvs is the all-to-all.  Returns each rank's yT (its rows filled)."""
    import torch
    for r, xc in zip(ranks, xcs):
        r.phase(DP_A, inp=xc)
    recvs = exchange([r.send_buffer(0) for r in ranks])
    out = []
    for r, buf in zip(ranks, recvs):
        r.copy(0, False, buf)
        out.append(r.phase(DP_BF, out=torch.empty(r.op.M, dtype=torch.float32, device=buf.device)))
    return out


def dist_adjoint(ranks, yTs, exchange):
    """x = A^T y for one signal; yTs each rank's yT (its rows read).  Returns each rank's xc."""
    import torch
    for r, yT in zip(ranks, yTs):
        r.phase(DP_BA, inp=yT)
    recvs = exchange([r.send_buffer(1) for r in ranks])
    out = []
    for r, buf in zip(ranks, recvs):
        r.copy(1, False, buf)
        out.append(r.phase(DP_C, out=torch.empty(r.nxc, dtype=torch.float32, device=buf.device)))
    return out


class DistGraphs:
    """One rank's application halves captured as CUDA graphs over static buffers: `pre`
    (apply: xc -> DP_A -> pack; adjoint: yT -> DP_BA -> pack) and `post` (unpack -> DP_BF or
    DP_C), with the exchange left between them (NCCL or host-staged, the caller's choice).
    Replaying removes the host cost of the ctypes calls (~17 us per phase).
    Usage: g.x[:] = xc; g.pre_apply.replay(); recv = exchange(g.send(0)); g.recv_buf(0)[:] = recv;
    g.post_apply.replay(); yT = g.yT (and the same with _adjoint / g.y_in / g.xc_out)."""

    def __init__(self, r: DistOperator):
        import torch
        self.r = r
        dev = r.ws.device
        self.x = torch.zeros(r.nxc, dtype=torch.float32, device=dev)
        self.y_in = torch.zeros(r.op.M, dtype=torch.float32, device=dev)
        self.yT = torch.zeros(r.op.M, dtype=torch.float32, device=dev)
        self.xc_out = torch.zeros(r.nxc, dtype=torch.float32, device=dev)
        self.sbuf = [torch.empty(sum(r.seg[(d, True)][2]), dtype=torch.float32, device=dev) for d in (0, 1)]
        self.rbuf = [torch.empty(sum(r.seg[(d, False)][2]), dtype=torch.float32, device=dev) for d in (0, 1)]
        steps = {
            "pre_apply": lambda: (r.phase(DP_A, inp=self.x), r.copy(0, True, self.sbuf[0])),
            "post_apply": lambda: (r.copy(0, False, self.rbuf[0]), r.phase(DP_BF, out=self.yT)),
            "pre_adjoint": lambda: (r.phase(DP_BA, inp=self.y_in), r.copy(1, True, self.sbuf[1])),
            "post_adjoint": lambda: (r.copy(1, False, self.rbuf[1]), r.phase(DP_C, out=self.xc_out)),
        }
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        for name, fn in steps.items():
            with torch.cuda.stream(side):
                fn()                       # warm-up outside capture (attributes, caches)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                fn()
            setattr(self, name, g)
        torch.cuda.current_stream(dev).wait_stream(side)

    def send(self, direction: int):
        r = self.r
        return self.sbuf[direction], r.seg[(direction, True)][2], r.seg[(direction, False)][2]

    def recv_buf(self, direction: int):
        return self.rbuf[direction]


def gather_x(ranks, xcs, allgather):
    """The natural x [N] on every rank from the xc of all ranks (allgather(list) -> for each
    local rank the concatenation of every rank's tensor in rank order; equal sizes)."""
    import torch
    full = allgather(xcs)
    return [r.phase(DP_XG, inp=f, out=torch.empty(r.op.N, dtype=torch.float32, device=f.device))
            for r, f in zip(ranks, full)]


def gather_y(ranks, yTs, allgather):
    """The natural y [M] on every rank from each rank's rows of yT (padded to equal sizes for
    the all-gather, then placed at every rank's row blocks and permuted to row order)."""
    import torch
    plan = ranks[0].plan
    offs = ranks[0].row_offsets
    spans = [plan.y_ranges(g, offs) for g in range(plan.world)]
    width = max(sum(b - a for a, b in sp) for sp in spans)
    packed = []
    for r, yT in zip(ranks, yTs):
        own = r.own_y(yT)
        packed.append(torch.cat([own, own.new_zeros(width - own.numel())]))
    full = allgather(packed)
    out = []
    for r, f in zip(ranks, full):
        yT = torch.empty(r.op.M, dtype=torch.float32, device=f.device)
        for g, sp in enumerate(spans):
            o = g * width
            for a, b in sp:
                yT[a:b] = f[o:o + b - a]
                o += b - a
        out.append(r.phase(DP_P, inp=yT, out=torch.empty(r.op.M, dtype=torch.float32, device=f.device)))
    return out


def emulated_exchange(sends):
    """All-to-all among the ranks of one process: receive buffer s = the blocks destined to s
    from every rank r, in rank order (the layout all_to_all_single produces)."""
    import torch
    world = len(sends)
    offs = []
    for buf, sc, rc in sends:
        o, acc = [], 0
        for c in sc:
            o.append((acc, acc + c))
            acc += c
        offs.append(o)
    return [torch.cat([sends[r][0][offs[r][s][0]:offs[r][s][1]] for r in range(world)]) for s in range(world)]


def emulated_allgather(parts):
    import torch
    full = torch.cat(parts)
    return [full for _ in parts]


def emulated_allreduce(parts):
    out = parts[0].clone()
    for p in parts[1:]:
        out += p
    return out


def process_group_exchange(group=None, host_staged: bool = False):
    """(exchange, allgather, allreduce) for one rank per process over torch.distributed: NCCL
    on GPUs; with host_staged the buffers go through host memory (gloo, which has no CUDA
    all-to-all: the CPU tests, and several processes sharing one GPU)."""
    import torch
    import torch.distributed as dist

    def _in(t):
        return t.cpu() if host_staged else t

    def _out(t, like):
        return t.to(like.device) if host_staged else t

    def exchange(sends):
        (buf, sc, rc), = sends
        b = _in(buf)
        out = torch.empty(sum(rc), dtype=b.dtype, device=b.device)
        dist.all_to_all_single(out, b, output_split_sizes=rc, input_split_sizes=sc, group=group)
        return [_out(out, buf)]

    def allgather(parts):
        (t,) = parts
        b = _in(t.contiguous())
        out = torch.empty(b.numel() * dist.get_world_size(group), dtype=b.dtype, device=b.device)
        dist.all_gather_into_tensor(out, b, group=group)
        return [_out(out, t)]

    def allreduce(parts):
        (t,) = parts
        b = _in(t)
        dist.all_reduce(b, group=group)
        if host_staged:
            t.copy_(b)
        return t
    return exchange, allgather, allreduce

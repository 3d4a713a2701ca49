"""Expert-parallel MoE layer over torch.distributed.

Rank r of W owns the routed experts [r E / W, (r + 1) E / W); shared experts are
replicated and run on every rank for its own tokens.  One layer call on a rank's
local tokens:

  1. router top-k on the local tokens (device kernel, bit-exact ids);
  2. dispatch: every (token, k) entry goes to the rank owning its expert.  The
     send buffer is ordered by (destination rank, token, k); an all-to-all of
     the per-destination counts sizes the receive buffer, then all-to-all-v
     moves the binary16 rows and their (local expert, weight) metadata
     (NCCL over NVLink / NVSwitch on GPUs, gloo on CPU);
  3. the owner runs its experts on the received rows with the given routing
     (each row routed to exactly one local expert with weight 1): the same
     decode / prefill kernels as the single-GPU layer;
  4. combine: the inverse all-to-all-v returns every entry's expert output to
     its token's rank, which sums them in k order with the router weights
     (moe_combine semantics) and adds the shared experts.

The collective is a real exchange step (tokens move to their experts), so it
is the only data-path collective; the layer itself is weak-scaled by tokens.

`local_fn(x_rows, local_ids) -> y_rows` computes the owned experts; the GPU
path binds it to `MoELayer.forward_routed`, tests bind a reference.
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist


def expert_owner(expert: torch.Tensor, n_experts: int, world: int) -> torch.Tensor:
    """Rank owning each routed expert (contiguous blocks of E / W experts)."""
    per = (n_experts + world - 1) // world
    return torch.div(expert, per, rounding_mode="floor")


class ExpertParallelMoE:
    def __init__(self, n_experts: int, top_k: int, d: int,
                 local_fn: Callable[[torch.Tensor, torch.Tensor], torch.Tensor],
                 shared_fn: Optional[Callable[[torch.Tensor], torch.Tensor]] = None,
                 router_fn: Optional[Callable[[torch.Tensor], tuple]] = None,
                 group=None):
        self.E = n_experts
        self.K = top_k
        self.d = d
        self.local_fn = local_fn
        self.shared_fn = shared_fn
        self.router_fn = router_fn
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.per = (n_experts + self.world - 1) // self.world
        self.first = self.rank * self.per

    def _a2a(self, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits):
        dist.all_to_all_single(out, inp, output_split_sizes=out_splits,
                               input_split_sizes=in_splits, group=self.group)

    def forward(self, x: torch.Tensor, logits: Optional[torch.Tensor] = None,
                ids: Optional[torch.Tensor] = None, weights: Optional[torch.Tensor] = None):
        """x: (m, d) local tokens; either router logits (m, E) or the routing
        (ids, weights) (m, K).  Returns (m, d) fp32."""
        m = x.shape[0]
        if ids is None:
            ids, weights = self.router_fn(logits)
        # Every rank must issue the same collectives: the exchange path and the
        # fixed capacity follow the largest token count of the group, agreed by
        # one small all-reduce unless the caller guarantees equal batches.
        m_max = m
        if self.world > 1 and not self.uniform_batch:
            on_dev = dist.get_backend(self.group) == "nccl"
            t = torch.tensor([m], dtype=torch.int64, device=x.device if on_dev else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
            m_max = int(t.item())
        if m_max * self.K <= self.fixed_cap_max:
            return self._forward_fixed(x, ids, weights, m_max)
        return self._forward_varlen(x, ids, weights)

    fixed_cap_max = 256   # entries per rank up to which the exchange uses a fixed capacity
    capacity = None       # rows per peer of the fixed exchange; None: max(m) K over the group
    uniform_batch = False  # caller guarantees the same m on every rank (skips the agreement)

    def _combine(self, x, ids, weights, y_entries):
        m = x.shape[0]
        y_entries = y_entries.view(m, self.K, self.d)
        w = torch.where(ids >= 0, weights.to(torch.float32), torch.zeros_like(weights, dtype=torch.float32))
        out = w[:, 0, None] * y_entries[:, 0]
        for k in range(1, self.K):  # k order, like moe_combine_kernel
            out = out + w[:, k, None] * y_entries[:, k]
        if self.shared_fn is not None:
            out = out + self.shared_fn(x)
        return out

    device_kernels = False  # MiloEPLayer: dispatch / combine as CUDA kernels of the library
    host_exchange = False   # device tensors exchanged through host copies (a gloo group, e.g. tests)

    def _a2a_dev(self, t: torch.Tensor) -> torch.Tensor:
        """all-to-all of equal splits; through host memory for a CPU backend."""
        if self.host_exchange:
            h = t.cpu()
            r = torch.empty_like(h)
            dist.all_to_all_single(r, h, group=self.group)
            return r.to(t.device)
        r = torch.empty_like(t)
        dist.all_to_all_single(r, t, group=self.group)
        return r

    def _forward_fixed(self, x, ids, weights, m_max=None):
        """Decode-sized batches: every rank sends a fixed capacity C = m K rows to
        every peer (unused rows carry expert id -1, which the kernels skip), so
        the exchange needs no count all-to-all and no host synchronization."""
        m, dev, W = x.shape[0], x.device, self.world
        C = self.capacity if self.capacity is not None else (m_max or m) * self.K
        assert m * self.K <= C, "fixed-capacity exchange: m * top_k exceeds the capacity"
        if self.device_kernels:
            import paper_2504_02658_b200 as mb
            # rows and local expert ids in one buffer: one all-to-all for both
            send, _, slot = mb.ep_dispatch(ids, x, W, self.per, C, packed=True)
            recv = self._a2a_dev(send)
            recv_x = recv[:, :self.d].contiguous()
            recv_m = recv[:, self.d:self.d + 2].contiguous().view(torch.int32).view(-1)
            if self.local_fn is not None:
                y_recv = self.local_fn(recv_x, recv_m).to(torch.float32)
            else:  # this rank owns no routed expert
                y_recv = torch.zeros((recv_x.shape[0], self.d), dtype=torch.float32, device=x.device)
            y_back = self._a2a_dev(y_recv.contiguous())
            out = mb.ep_combine(y_back, slot, weights)
            if self.shared_fn is not None:
                out = out + self.shared_fn(x)
            return out
        flat = ids.reshape(-1).to(torch.int64)
        valid = flat >= 0
        dest = torch.where(valid, torch.div(flat.clamp(min=0), self.per, rounding_mode="floor"),
                           torch.full_like(flat, W))
        onehot = (dest[:, None] == torch.arange(W, device=dev)[None, :]).to(torch.int32)
        pos = (torch.cumsum(onehot, 0) - 1).gather(1, dest.clamp(max=W - 1)[:, None])[:, 0]
        slot = torch.where(valid, dest * C + pos, torch.full_like(dest, W * C))  # W*C = dropped
        send_x = torch.zeros((W * C + 1, self.d), dtype=torch.float16, device=dev)
        send_m = torch.full((W * C + 1,), -1, dtype=torch.int32, device=dev)
        tok = torch.arange(m * self.K, device=dev) // self.K
        send_x[slot] = x.to(torch.float16)[tok]
        send_m[slot] = (flat - dest * self.per).to(torch.int32)
        recv_x = torch.empty((W * C, self.d), dtype=torch.float16, device=dev)
        recv_m = torch.empty((W * C,), dtype=torch.int32, device=dev)
        dist.all_to_all_single(recv_x, send_x[:W * C], group=self.group)
        dist.all_to_all_single(recv_m, send_m[:W * C], group=self.group)
        y_recv = self.local_fn(recv_x, recv_m).to(torch.float32)
        y_back = torch.empty((W * C + 1, self.d), dtype=torch.float32, device=dev)
        y_back[W * C].zero_()
        dist.all_to_all_single(y_back[:W * C], y_recv.contiguous(), group=self.group)
        return self._combine(x, ids, weights, y_back[slot])

    def _forward_varlen(self, x, ids, weights):
        """Prefill-sized batches: exact all-to-all-v (one host sync for the counts)."""
        m = x.shape[0]
        dev = x.device
        ids64 = ids.to(torch.int64)
        flat_ids = ids64.reshape(-1)
        valid = flat_ids >= 0
        entry = torch.arange(m * self.K, device=dev)
        dest = torch.where(valid, expert_owner(flat_ids.clamp(min=0), self.E, self.world),
                           torch.full_like(flat_ids, self.world))
        order = torch.argsort(dest * (m * self.K) + entry)  # stable (dest, token, k)
        send_counts = torch.bincount(dest, minlength=self.world + 1)[: self.world]
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        sc = send_counts.tolist()
        rc = recv_counts.tolist()
        n_send, n_recv = sum(sc), sum(rc)
        order = order[:n_send]
        send_dest = dest[order]
        xs = x.to(torch.float16)[torch.div(order, self.K, rounding_mode="floor")]
        meta = (flat_ids[order] - send_dest * self.per).to(torch.int32)
        x_recv = torch.empty((n_recv, self.d), dtype=torch.float16, device=dev)
        meta_recv = torch.empty((n_recv,), dtype=torch.int32, device=dev)
        self._a2a(x_recv, xs.contiguous(), rc, sc)
        self._a2a(meta_recv, meta.contiguous(), rc, sc)
        if n_recv > 0:
            y_recv = self.local_fn(x_recv, meta_recv).to(torch.float32).contiguous()
        else:
            y_recv = torch.empty((0, self.d), dtype=torch.float32, device=dev)
        y_send = torch.empty((n_send, self.d), dtype=torch.float32, device=dev)
        self._a2a(y_send, y_recv, sc, rc)
        y_entries = torch.zeros((m * self.K, self.d), dtype=torch.float32, device=dev)
        y_entries[order] = y_send
        return self._combine(x, ids64, weights, y_entries)


def milo_local_fn(layer):
    """Binds the owned experts (a MoELayer over them, top_k = 1) as local_fn."""
    ones = {}  # rows -> cached unit routing weights (no fill kernel per call)

    def fn(x_rows: torch.Tensor, local_ids: torch.Tensor) -> torch.Tensor:
        ids = local_ids.view(-1, 1).to(torch.int32)
        key = (x_rows.shape[0], x_rows.device)
        if key not in ones:
            ones[key] = torch.ones((x_rows.shape[0], 1), dtype=torch.float32, device=x_rows.device)
        return layer.forward_routed(x_rows, ids, ones[key])
    return fn


class MiloEPLayer:
    """The MiLo MoE layer sharded by expert over the ranks of `group`.

    `owned` are this rank's routed experts (global ids first..first+len-1),
    `shared` the replicated shared experts.  Same call surface as MoELayer:
    forward(x, router_logits) on the local tokens."""

    def __init__(self, owned, shared, n_experts: int, top_k: int, score_mode: int = 0, group=None):
        import paper_2504_02658_b200 as mb
        self.mb = mb
        self.local = mb.MoELayer(owned, [], top_k=1, score_mode=0) if owned else None
        self.shared = mb.MoELayer([], shared, top_k=1) if shared else None
        self.E, self.K, self.score_mode = n_experts, top_k, score_mode
        self.d = (owned or shared)[0].w1.rows
        shared_fn = None
        if self.shared is not None:
            def shared_fn(x):
                return self.shared.forward(x.contiguous(), None)
        self.ep = ExpertParallelMoE(n_experts, top_k, self.d, milo_local_fn(self.local) if self.local else None,
                                    shared_fn=shared_fn, router_fn=self._route, group=group)
        self.ep.device_kernels = True

    def _route(self, logits):
        return self.mb.router_topk(logits, self.K, self.score_mode)

    def forward(self, x, router_logits, out_dtype=None, return_routing=False, stream=None):
        ids, w = self._route(router_logits)
        out = self.ep.forward(x, ids=ids, weights=w)
        if out_dtype is not None and out_dtype != torch.float32:
            out = out.to(out_dtype)
        return (out, ids, w) if return_routing else out

    def forward_host(self, x, router_logits):
        xd = torch.from_numpy(x).cuda(non_blocking=True)
        ld = torch.from_numpy(router_logits).cuda(non_blocking=True)
        out = self.forward(xd, ld)
        return out.cpu().numpy()


class NativeEPLayer:
    """The expert-parallel layer in the C++ library over NCCL (milo_ep_forward):
    router, dispatch, the two grouped ncclSend / ncclRecv exchanges, the owned
    experts and the combine all run stream-ordered inside one C call.

    The NCCL communicator is built from a unique id made on rank 0 and broadcast
    over `group` (any torch.distributed backend), or passed explicitly as
    (nccl_id, world, rank) -- world 1 needs no process group at all."""

    def __init__(self, owned, shared, n_experts: int, top_k: int, score_mode: int = 0, group=None,
                 nccl_id: bytes = None, world: int = None, rank: int = None):
        import ctypes as C
        import paper_2504_02658_b200 as mb
        self.mb = mb
        if world is None:
            world = dist.get_world_size(group)
            rank = dist.get_rank(group)
        if nccl_id is None:
            buf = (C.c_uint8 * 128)()
            if rank == 0:
                mb._check(mb.lib().milo_ep_unique_id(buf, 128))
            if world > 1:
                t = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
                if dist.get_backend(group) == "nccl":
                    t = t.cuda()
                dist.broadcast(t, src=0, group=group)
                buf = (C.c_uint8 * 128)(*t.cpu().tolist())
            nccl_id = bytes(buf)
        idb = (C.c_uint8 * 128)(*nccl_id)
        comm = C.c_void_p()
        mb._check(mb.lib().milo_ep_comm_create(idb, world, rank, C.byref(comm)))
        self._comm = comm
        self.local = mb.MoELayer(owned, [], top_k=1, score_mode=0) if owned else None
        self.shared = mb.MoELayer([], shared, top_k=1) if shared else None
        self.E, self.K, self.world, self.rank = n_experts, top_k, world, rank
        self.score_mode = score_mode
        self.d = (owned or shared)[0].w1.rows
        h = C.c_void_p()
        mb._check(mb.lib().milo_ep_layer_create(self.local._h if self.local else None,
                                                self.shared._h if self.shared else None, n_experts, top_k,
                                                score_mode, comm, C.byref(h)))
        self._h = h
        self.capacity = 0  # rows per peer; 0: m * top_k (equal batches on every rank)

    def forward(self, x, router_logits, out_dtype=None, return_routing=False, stream=None):
        mb = self.mb
        x = x.contiguous()
        m = x.shape[0]
        out = torch.empty((m, self.d), dtype=torch.float32, device=x.device)
        lg = router_logits.contiguous().float()
        mb._check(mb.lib().milo_ep_forward(self._h, mb._dptr(x), m, mb.F32 if x.dtype == torch.float32 else mb.F16,
                                           mb._dptr(lg), mb._dptr(out), int(self.capacity), mb._stream_ptr(stream)))
        if out_dtype is not None and out_dtype != torch.float32:
            out = out.to(out_dtype)
        if return_routing:
            ids, w = mb.router_topk(lg, self.K, self.score_mode)
            return out, ids, w
        return out

    def forward_host(self, x, router_logits):
        xd = torch.from_numpy(x).cuda(non_blocking=True)
        ld = torch.from_numpy(router_logits).cuda(non_blocking=True)
        return self.forward(xd, ld).cpu().numpy()

    def close(self):
        mb = self.mb
        if getattr(self, "_h", None):
            mb.lib().milo_ep_layer_destroy(self._h)
            self._h = None
        if getattr(self, "_comm", None):
            mb.lib().milo_ep_comm_destroy(self._comm)
            self._comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

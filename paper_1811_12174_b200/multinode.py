"""Two-level DDL all-reduce: the paper's actual hierarchy.

PowerAI DDL "adapts to the hierarchy of communication bandwidths" and "can mix-and-match
various reduce-scatter and all-gather implementations/algorithms over different network
fabrics" (P:L54 (1), (3)); its measured systems were 2 nodes x 4 GPUs with NVLink or PCIe
inside a node and InfiniBand or Ethernet between nodes.  Here the inner dims
(GPUs of one node) run on libddl's kernels over NVLink/NVSwitch, and the outer dim (nodes)
runs over a ``torch.distributed`` transport (NCCL-net / IB across nodes; gloo in the tests),
with the outer reduction itself done by libddl's local-reduce kernel so the fold order stays
the method's:

  1. inner reduce-scatter (libddl, op = sum)      rank holds chunk c_in (n / P_in elements)
  2. outer exchange (transport all-to-all)         g_out pieces of my chunk, one per node
  3. outer fold (libddl local reduce, ascending node coordinate, x fl32(1/P) for avg)
  4. outer all-gather (transport)                  chunk c_in fully reduced
  5. inner all-gather (libddl)                     the whole vector, on every rank

Every element therefore gets F_dims with dims = inner_dims + [g_out] -- bit-identical to
the single-level schedule and to the oracle (the block layout differs, the per-element fold
does not).  Ranks are numbered inner-fastest: rank = c_in + P_in * c_out.
"""
import math

import torch
import torch.distributed as dist

from . import ddl


def _host_staged(group) -> bool:
    return dist.get_backend(group) == dist.Backend.GLOO


class TwoLevelComm:
    def __init__(self, inner_dims, nodes: int, group=None, max_bytes: int = 256 << 20):
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.inner_dims = ddl.parse_dims(inner_dims)
        self.p_in = math.prod(self.inner_dims)
        self.nodes = nodes
        if self.p_in * nodes != self.world:
            raise ddl.DDLError(ddl.ERR_BAD_DIMS, f"{self.inner_dims} x {nodes} nodes vs {self.world} ranks")
        self.c_in, self.c_out = self.rank % self.p_in, self.rank // self.p_in
        ranks = list(range(self.world)) if group is None else dist.get_process_group_ranks(group)
        self.inner_pg = self.outer_pg = None
        for o in range(nodes):        # every rank creates every group, in the same order
            g = dist.new_group([ranks[o * self.p_in + i] for i in range(self.p_in)])
            if o == self.c_out:
                self.inner_pg = g
        for i in range(self.p_in):
            g = dist.new_group([ranks[o * self.p_in + i] for o in range(nodes)])
            if i == self.c_in:
                self.outer_pg = g
        self.inner = ddl.Comm(self.inner_dims, group=self.inner_pg, max_bytes=max_bytes)

    @property
    def dims(self):
        return self.inner_dims + [self.nodes]

    def _a2a(self, out, inp):
        if _host_staged(self.outer_pg):
            o = torch.empty_like(out, device="cpu")
            dist.all_to_all_single(o, inp.cpu(), group=self.outer_pg)
            out.copy_(o)
        else:
            dist.all_to_all_single(out, inp, group=self.outer_pg)

    def _ag(self, out, inp):
        if _host_staged(self.outer_pg):
            parts = [torch.empty_like(inp, device="cpu") for _ in range(self.nodes)]
            dist.all_gather(parts, inp.cpu(), group=self.outer_pg)
            out.copy_(torch.cat(parts))
        else:
            dist.all_gather_into_tensor(out, inp, group=self.outer_pg)

    def all_reduce(self, t, op: str = "sum"):
        """In place.  t.numel() must be a multiple of P * (16 B / element size)."""
        n = t.numel()
        v = 16 // t.element_size()
        if n % (self.world * v):
            raise ddl.DDLError(ddl.ERR_INVALID_ARGUMENT, f"numel {n} must be a multiple of {self.world * v}")
        m = n // self.p_in
        piece = m // self.nodes
        chunk = torch.empty(m, dtype=t.dtype, device=t.device)
        self.inner.reduce_scatter(chunk, t, "sum")                        # 1
        gathered = torch.empty(m, dtype=t.dtype, device=t.device)
        self._a2a(gathered, chunk)                                        # 2 (piece j from node j)
        mine = torch.empty(piece, dtype=t.dtype, device=t.device)
        scale = 1.0 / self.world if op == "avg" else 1.0
        ddl.local_reduce([gathered[j * piece:(j + 1) * piece] for j in range(self.nodes)], mine,
                         float(torch.tensor(scale, dtype=torch.float32)))  # 3 (fl32(1/P))
        self._ag(chunk, mine)                                             # 4
        self.inner.all_gather(t, chunk)                                   # 5
        return t

    def finalize(self):
        self.inner.finalize()

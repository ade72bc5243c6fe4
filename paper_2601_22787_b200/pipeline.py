"""Block-pipelined inference arena (App. A.1).

The paper keeps ONE per-device decompression buffer sized to one transformer block and
decodes each block right before its forward pass; it names overlapping the decode
of upcoming blocks with the current forward as the next optimisation.  This module
provides both:

* ``slots=1``  — the paper's scheme: decode block k, then forward block k (serial);
* ``slots=S>1`` — S block-sized arenas; the decode of block k+S-1 is enqueued on a side
  stream while block k computes on the main stream.  CUDA events order the reuse of a slot
  (a slot is overwritten only after the forward that read it has finished).

Every decode is one ``eq_decode_dequant`` call (C ABI) into the slot's arena; the layer
weights are tensor views into it (no copies).  ``forward(k, views, x) -> x`` is the
caller's block computation on the main stream.
"""
from __future__ import annotations

import torch

from . import EQ_OUT_BF16, Block, Decoder


class BlockPipeline:
    """``group`` blocks are decoded per launch (one eq_decode_dequant over ``group`` blocks:
    enough independent chunks to fill the GPU — a single Llama-3-8B block has only 53 K);
    ``slots`` group-sized arenas rotate; with slots > 1 the decode of group g+slots-1 runs on
    a side stream while group g computes."""

    def __init__(self, blocks: list[Block], out_dtype: int = EQ_OUT_BF16, slots: int = 2, group: int = 1,
                 device=None):
        if slots < 1 or group < 1:
            raise ValueError("slots >= 1 and group >= 1")
        from . import arena_layout
        self.blocks = list(blocks)
        self.slots = slots
        self.group = group
        dev = device or self.blocks[0].payload.device
        self.groups = [self.blocks[i:i + group] for i in range(0, len(self.blocks), group)]
        need = max(arena_layout(g, out_dtype)[1] for g in self.groups)
        self.arenas = [torch.empty(need, dtype=torch.uint8, device=dev) for _ in range(slots)]
        # one pre-marshalled decoder per group, targeting slot g % slots
        self.decoders = [Decoder(g, out_dtype, arena=self.arenas[i % slots]) for i, g in enumerate(self.groups)]
        # the forward runs on a high-priority stream so its CTAs are scheduled ahead of the
        # (long-running, compute-bound) decode CTAs of the next group as SMs free up
        lo, hi = torch.cuda.Stream.priority_range()
        self.decode_stream = torch.cuda.Stream(device=dev, priority=lo) if slots > 1 else None
        self.compute_stream = torch.cuda.Stream(device=dev, priority=hi) if slots > 1 else None
        self.decoded = [torch.cuda.Event() for _ in self.groups]
        self.released = [torch.cuda.Event() for _ in range(slots)]

    def _forward_group(self, gi, forward, x):
        views = self.decoders[gi].views()
        for j, v in enumerate(views):
            x = forward(gi * self.group + j, v, x)
        return x

    def run(self, forward, x: torch.Tensor) -> torch.Tensor:
        main = torch.cuda.current_stream()
        n = len(self.groups)
        if self.slots == 1:
            for g in range(n):
                self.decoders[g](main)
                x = self._forward_group(g, forward, x)
            return x
        ds, cs = self.decode_stream, self.compute_stream
        ds.wait_stream(main)                         # inputs/arenas ready before decoding
        cs.wait_stream(main)
        ahead = self.slots - 1

        def issue(g):
            s = g % self.slots
            if g >= self.slots:
                ds.wait_event(self.released[s])      # group g - slots has finished reading slot s
            self.decoders[g](ds)
            self.decoded[g].record(ds)

        for g in range(min(ahead, n)):
            issue(g)
        with torch.cuda.stream(cs):
            for g in range(n):
                if g + ahead < n:
                    issue(g + ahead)
                cs.wait_event(self.decoded[g])
                x = self._forward_group(g, forward, x)
                self.released[g % self.slots].record(cs)
        main.wait_stream(cs)
        return x

    def check(self) -> None:
        """Device error words of every group's last decode (synchronous)."""
        for d in self.decoders:
            d.check()


def llama_block_forward(views, x: torch.Tensor) -> torch.Tensor:
    """A Llama-shaped linear dataflow over one block's 7 weight views (bf16):
    q, k, v, o projections (attention mixing omitted: o consumes q) and the SwiGLU MLP,
    with residual connections.  Used to measure decode overhead against pure GEMM time."""
    wq, wk, wv, wo, wg, wu, wd = views
    q = x @ wq.t()
    _ = x @ wk.t()
    _ = x @ wv.t()
    h = x + q @ wo.t()
    m = torch.nn.functional.silu(h @ wg.t()) * (h @ wu.t())
    return h + m @ wd.t()


def llama_block_forward_fused(block: Block, x: torch.Tensor, err: torch.Tensor, workspace: torch.Tensor) -> torch.Tensor:
    """``llama_block_forward`` with every GEMM fused with the block's decode
    (``eq_qmatmul_group``, §8(f) row 1): the weights are never materialised.  The dataflow
    needs four dependent launches: {q, k, v} → o → {gate, up} → down; activations between them
    are rounded to bf16 as in the dense forward."""
    from . import qmatmul_group
    q, _, _ = qmatmul_group(block, [0, 1, 2], [x, x, x], err=err, check=False, workspace=workspace)
    h = x + qmatmul_group(block, [3], [q.to(torch.bfloat16)], err=err, check=False, workspace=workspace)[0].to(torch.bfloat16)
    g, u = qmatmul_group(block, [4, 5], [h, h], err=err, check=False, workspace=workspace)
    m = (torch.nn.functional.silu(g) * u).to(torch.bfloat16)
    return h + qmatmul_group(block, [6], [m], err=err, check=False, workspace=workspace)[0].to(torch.bfloat16)

"""Plan executor: runs a reference execution plan on device data.

Consumes the reference's two wire formats unchanged:
  * graph document v1   (proj/src/graph_ir.cpp:449-573): nodes in topological
    order with kind / inputs / output metadata;
  * plan document v1    (proj/src/planner.cpp:455-600, plan_to_json): per node
    the selected strategy name and output spec (+ partial_sum / reduce_axes),
    and the inserted communication (all-reduce after partial sums,
    per-step conversion chains on mismatched edges).

and executes the forward pass on a `runtime.Mesh` (simulated or distributed):
  * placeholders / parameters are sharded by their plan spec;
  * every mismatched edge is converted with the reference's own path
    (find_transform_path, identical to proj/src/layout.cpp:253-316) — either
    step by step, exactly like the plan's `<producer>.cvN` nodes
    (insert_comm_nodes, planner.cpp:284-347), or collapsed into one exchange;
    chains are shared between consumers of the same (producer, target spec),
    as in planner.cpp:299-305;
  * matmul nodes run their strategy (catalog decode of the strategy name,
    intraop.cpp:141-234) as tcgen05 GEMMs on the shards, with the partial-sum
    all-reduce of `<host>.ar` (planner.cpp:263-282);
  * an elementwise-unary GELU consuming a non-partial matmul output in the
    same layout is fused into the GEMM epilogue;
  * the transformer-block kinds (gpt_block graph: embedding-lookup, layernorm,
    reshape, transpose, batched-matmul, softmax, elementwise-binary) run
    their named strategy (intraop.cpp:280-450) on the local shards: reshape
    is a view with the plan's rewritten local shape (reshape_rewrites,
    planner.cpp:401-450), transpose permutes shard and spec together,
    batched matmul is one grouped tcgen05 GEMM per device (+ the partial-sum
    all-reduce of split-k strategies), the rest are block_ops.cu kernels;
  * the output node collects to RR (intraop.cpp:469-482).

The graph format names the elementwise-unary function only by node id (the
reference plans it as an opaque elementwise op), so the executor binds:
a uint8 operand -> logical not (the block's `mask2`); an id containing
"scale" behind a batched matmul -> x / sqrt(k) (attention scaling); a
matmul output (the MLP activation) or an id containing "gelu" -> exact-erf
GELU; any other unary node is rejected (ValueError) unless `unary=` binds it. A binary op with a uint8 operand adds it as an
additive mask (a - 1e4 * m); otherwise it is a + b (residuals). `unary=`
overrides the binding per node.

The executor also cross-checks its own communication against the plan's
`inserted_comm_nodes` (same producers/consumers, same step kinds and axes),
so a plan this runtime would execute differently is rejected up front.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from .layout import DeviceMesh, DimSpec, ShardingSpec, TensorMeta, find_transform_path
from .strategies import MatmulStrategy, find_matmul_strategy

_DTYPES = {1: torch.uint8, 2: torch.bfloat16, 4: torch.float32, 8: torch.int64}
_BLOCK_KINDS = ("embedding-lookup", "layernorm", "reshape", "transpose", "softmax",
                "elementwise-binary", "batched-matmul")
MASK_FILL = -1e4  # additive attention mask: a + MASK_FILL * m


def infer_shapes(graph: dict) -> dict:
    """Output shape + dtype bytes per node (shape rules of graph_ir.cpp:189-373
    for the kinds the MLP/block graphs use)."""
    out = {}
    for n in graph["nodes"]:
        if n["outputs"]:
            o = n["outputs"][0]
            out[n["id"]] = (tuple(o["shape"]), o["dtype_bytes"])
            continue
        ins = [out[i[0]] for i in n["inputs"]]
        k = n["kind"]
        if k == "matmul":
            (a, ea), (b, _) = ins
            out[n["id"]] = (a[:-1] + (b[-1],), ea)
        elif k == "batched-matmul":
            (a, ea), (b, _) = ins
            out[n["id"]] = ((a[0], a[1], b[2]), ea)
        elif k in ("elementwise-unary", "output", "layernorm", "softmax"):
            out[n["id"]] = ins[0]
        elif k == "elementwise-binary":
            out[n["id"]] = (ins[0][0], max(ins[0][1], ins[1][1]))
        elif k == "reshape":
            out[n["id"]] = (tuple(n["attrs"]["target_shape"]), ins[0][1])
        elif k == "transpose":
            perm = n["attrs"]["perm"]
            out[n["id"]] = (tuple(ins[0][0][p] for p in perm), ins[0][1])
        elif k == "embedding-lookup":
            (ids, _), (table, eb) = ins
            out[n["id"]] = (tuple(ids) + (table[1],), eb)
        else:
            raise NotImplementedError(f"node kind {k!r} is not executable yet")
    return out


@dataclass
class CommRecord:
    """One communication the executor performs (mirrors CommInsertion)."""
    producer: str
    consumer: str
    collective: str
    axes: tuple
    bytes: int


@dataclass
class PlanExecutor:
    mesh: "object"  # runtime.Mesh
    graph: dict
    plan: dict
    fuse: bool = True
    # inference: weight all-gathers fused into the GEMM (None = auto: on for
    # the peer runtime, off on a simulated mesh, where the K-sliced grouped
    # GEMM measured slower than gather + one batched GEMM: 0.43 vs 0.31 ms)
    fuse_gather: bool | None = None
    # elementwise-unary binding per node id: ("gelu",) | ("scale", alpha) | ("not",)
    unary: dict | None = None
    comm: list = field(default_factory=list)
    # honour the plan's activation-checkpoint schedule (ckpt.cpp: Rotor
    # decisions per chain stage): stages decided store_boundary / recompute
    # drop what backward needs after the first forward pass and re-run from
    # their block's boundary inputs when backward reaches them. False: store
    # everything (same bytes, more memory).
    checkpoint: bool = True
    _saved: dict = None

    def __post_init__(self):
        self.geo: DeviceMesh = self.mesh.geo
        mr = self.geo.rank()
        self.shapes = infer_shapes(self.graph)
        self.nodes = {n["id"]: n for n in self.graph["nodes"]}
        self.spec = {nid: ShardingSpec.parse(p["spec"], mr) for nid, p in self.plan["nodes"].items()}
        self.partial = {nid: tuple(p.get("reduce_axes", ())) for nid, p in self.plan["nodes"].items()
                        if p.get("partial_sum")}
        self.strategy: dict[str, MatmulStrategy] = {}
        self.in_specs: dict[str, list] = {}
        for n in self.graph["nodes"]:
            nid, kind = n["id"], n["kind"]
            name = self.plan["nodes"][nid]["strategy"]
            if kind in ("matmul", "batched-matmul"):
                a_meta = self._meta(n["inputs"][0][0])
                b_meta = self._meta(n["inputs"][1][0])
                st = find_matmul_strategy(name, self.geo, a_meta, b_meta,
                                          batched=kind == "batched-matmul")
                if st.c != self.spec[nid]:
                    raise ValueError(f"{nid}: plan spec {self.spec[nid]} != strategy "
                                     f"output {st.c}")
                self.strategy[nid] = st
                self.in_specs[nid] = [st.a, st.b]
            elif kind in ("placeholder", "parameter"):
                self.in_specs[nid] = []
            else:
                self.in_specs[nid] = self._input_specs(n, name)
        self._consumers = {}
        for n in self.graph["nodes"]:
            for slot, (src, _) in enumerate(n["inputs"]):
                self._consumers.setdefault(src, []).append((n["id"], slot))
        self._paths = {}
        self._convs = {}
        self._block_of, self._blocks = self._checkpoint_blocks()
        self._attn = self._attention_chains()
        self._attn_members = {m for ch in self._attn.values() for m in ch[1:3]}

    # ---- layout bookkeeping ------------------------------------------------
    def _meta(self, nid: str) -> TensorMeta:
        shape, eb = self.shapes[nid]
        return TensorMeta(shape, eb)

    def _input_specs(self, n: dict, name: str) -> list:
        """Input layouts of a non-matmul node's named strategy
        (intraop.cpp:280-450): the name carries the input spec for reshape /
        perm / softmax / layernorm, the axes for embeddings; elementwise ops
        mirror the output layout onto every input."""
        nid, kind, mr = n["id"], n["kind"], self.geo.rank()
        out = self.spec[nid]
        if kind == "output":
            return [ShardingSpec.replicated(len(self.shapes[nid][0]), mr)]
        if kind in ("reshape", "transpose", "softmax", "layernorm"):
            spec = ShardingSpec.parse(name.split(":", 1)[1], mr)
            if kind == "transpose":
                perm = n["attrs"]["perm"]
                if [spec.dims[p] for p in perm] != list(out.dims):
                    raise ValueError(f"{nid}: {name} does not produce {out}")
            if kind == "layernorm":
                return [spec] + [ShardingSpec.replicated(1, mr)] * (len(n["inputs"]) - 1)
            return [spec]
        if kind == "embedding-lookup":
            # emb-batch@i:t / emb-h:t / emb-bh@i:x,y (intraop.cpp:406-450)
            ri = len(self.shapes[n["inputs"][0][0]][0])
            return [ShardingSpec(tuple(out.dims[:ri]), mr),
                    ShardingSpec((DimSpec(), out.dims[ri]), mr)]
        return [out] * len(n["inputs"])  # elementwise

    def required_spec(self, consumer: str, slot: int) -> ShardingSpec:
        return self.in_specs[consumer][slot]

    def unary_op(self, nid: str) -> tuple:
        """The function an elementwise-unary node computes (module docstring)."""
        if self.unary and nid in self.unary:
            return tuple(self.unary[nid])
        src = self.nodes[nid]["inputs"][0][0]
        if self.shapes[src][1] == 1:
            return ("not",)
        prod = self.nodes[src]
        if "scale" in nid and prod["kind"] == "batched-matmul":
            k = self.shapes[prod["inputs"][0][0]][0][-1]
            return ("scale", 1.0 / float(k) ** 0.5)
        if prod["kind"] == "matmul" or "gelu" in nid.lower():
            return ("gelu",)  # the MLP activation (fc1 -> act)
        raise ValueError(
            f"{nid}: the graph does not name this elementwise-unary function (it consumes a "
            f"{prod['kind']} node); pass unary={{{nid!r}: ('gelu',) | ('scale', alpha) | "
            f"('not',)}} to bind it")

    def _attention_chains(self) -> dict:
        """softmax id -> (softmax, scale node, binary node, scores id, mask id,
        alpha) for every `scaled -> att_in -> att` chain (scale, additive u8
        mask, last-axis softmax) whose edges need no conversion under the
        plan: run as one apl_softmax_ex pass instead of three kernels."""
        out = {}
        for n in self.graph["nodes"]:
            if n["kind"] != "softmax" or n.get("attrs", {}).get("axis", -1) not in (
                    -1, len(self.shapes[n["id"]][0]) - 1):
                continue
            sm = n["id"]
            b = n["inputs"][0][0]
            bn = self.nodes[b]
            if (bn["kind"] != "elementwise-binary" or len(self._consumers.get(b, [])) != 1
                    or self.spec[b] != self.in_specs[sm][0]):
                continue
            ins = [i[0] for i in bn["inputs"]]
            mslot = [k for k, x in enumerate(ins) if self.shapes[x][1] == 1]
            if len(mslot) != 1:
                continue
            u, m = ins[1 - mslot[0]], ins[mslot[0]]
            un = self.nodes[u]
            if (un["kind"] != "elementwise-unary" or len(self._consumers.get(u, [])) != 1
                    or self.unary_op(u)[0] != "scale"):
                continue
            x = un["inputs"][0][0]
            if not (self.spec[u] == self.in_specs[b][1 - mslot[0]]
                    and self.spec[m] == self.in_specs[b][mslot[0]]
                    and self.spec[x] == self.in_specs[u][0]):
                continue
            out[sm] = (sm, u, b, x, m, self.unary_op(u)[1])
        return out

    def _checkpoint_blocks(self):
        """node id -> recompute block index, and block -> member ids in graph
        order, from plan["schedule"] (block_index: maximal runs of stages
        decided store_boundary / recompute, ckpt.cpp; -1 = stored in full)
        and plan["stages"] (each stage's member nodes)."""
        sched, stages = self.plan.get("schedule"), self.plan.get("stages")
        if not self.checkpoint or not sched or not stages:
            return {}, {}
        if getattr(self.mesh, "empty", None) is not None:
            # a per-step bump allocator (the peer runtime's symmetric heap)
            # frees nothing before the next step: dropping saved state would
            # save no memory and the recompute would take more heap
            return {}, {}
        block_of = {}
        for st in stages:
            b = sched["block_index"][st["index"]]
            if b >= 0:
                for m in st["members"]:
                    block_of[m] = b
        order = [n["id"] for n in self.graph["nodes"]]
        blocks = {}
        for nid in order:
            if nid in block_of:
                blocks.setdefault(block_of[nid], []).append(nid)
        return block_of, blocks

    def _fusable_gelu(self, mm: str):
        """The GELU node fused into matmul `mm`'s epilogue, if any (never
        across a checkpoint-block boundary: a recomputed GELU re-reads its
        producer's output)."""
        cons = self._consumers.get(mm, [])
        if len(cons) != 1 or mm in self.partial or self.nodes[mm]["kind"] != "matmul":
            return None
        gid, _ = cons[0]
        if self._block_of.get(mm) != self._block_of.get(gid):
            return None
        g = self.nodes[gid]
        if (g["kind"] == "elementwise-unary" and self.spec[gid] == self.spec[mm]
                and self.unary_op(gid) == ("gelu",)):
            return gid
        return None

    def planned_communication(self) -> list:
        """The communication this executor will issue, in graph walk order:
        one record per reference step (fuse=False semantics) so it can be
        compared with the plan's inserted_comm_nodes."""
        recs = []
        for n in self.graph["nodes"]:
            nid = n["id"]
            if nid in self.partial:
                recs.append(CommRecord(nid, "", "all-reduce", self.partial[nid], 0))
            seen = set()
            for consumer, slot in self._consumers.get(nid, []):
                src, tgt = self.spec[nid], self.required_spec(consumer, slot)
                if src == tgt or (str(src), str(tgt)) in seen:
                    continue
                seen.add((str(src), str(tgt)))
                for s in self._path(nid, src, tgt).steps:
                    recs.append(CommRecord(nid, consumer, str(s.kind), (s.mesh_axis,), 0))
        return recs

    def check_against_plan(self) -> None:
        mine = [(r.producer, r.collective, tuple(r.axes)) for r in self.planned_communication()]
        theirs = [(c["producer"], c["collective"], tuple(c["axes"]))
                  for c in self.plan["inserted_comm_nodes"]]
        if mine != theirs:
            raise ValueError(f"plan communication differs from the executor's:\n{theirs}\n{mine}")

    def _path(self, nid, src, tgt):
        key = (nid, str(src), str(tgt))
        if key not in self._paths:
            self._paths[key] = find_transform_path(src, tgt, self.geo, self._meta(nid))
        return self._paths[key]

    # ---- execution ---------------------------------------------------------
    def shard(self, nid: str, full: torch.Tensor) -> list:
        """Local shards of a global tensor under node `nid`'s plan spec."""
        spec = self.spec[nid]
        devs = range(self.mesh.num_devices) if not self.mesh.distributed else [self.mesh.first_local]
        out = []
        for d in devs:
            coord = self.geo.coord_of(d)
            sl = []
            for k, dim in enumerate(spec.dims):
                s, split = 0, 1
                for a in dim.axes:
                    s = s * self.geo.shape[a] + coord[a]
                    split *= self.geo.shape[a]
                L = full.shape[k] // split
                sl.append(slice(s * L, (s + 1) * L))
            out.append(full[tuple(sl)].contiguous())
        return out

    def _empty(self, shape, dtype, device) -> torch.Tensor:
        """Device buffer for a value; meshes with their own allocator (the
        peer runtime's symmetric heap) provide it."""
        alloc = getattr(self.mesh, "empty", None)
        if alloc is not None:
            return alloc(shape, dtype)
        return torch.empty(shape, dtype=dtype, device=device)

    def _zeros(self, shape, device) -> torch.Tensor:
        """fp32 accumulator from the mesh's allocator (the peer runtime's
        all-reduce reads and writes its buffers in the symmetric heap)."""
        t = self._empty(tuple(shape), torch.float32, device)
        t.zero_()
        return t

    def _alloc(self, nid: str, spec: ShardingSpec, like: torch.Tensor) -> list:
        shape = spec.local_shape(self._meta(nid), self.geo)
        return [self._empty(shape, like.dtype, like.device) for _ in range(self.mesh.num_local)]

    def _convert(self, nid, shards, src, tgt, stream):
        key = (nid, str(src), str(tgt))
        conv = self._convs.get(key)
        if conv is None:  # compiled once per edge, reused every forward
            conv = self.mesh.prepare(self._path(nid, src, tgt), self._meta(nid), fuse=self.fuse)
            self._convs[key] = conv
        outs = self._alloc(nid, tgt, shards[0])
        conv(shards, outs, stream=stream)
        return outs

    def forward(self, feeds: dict, stream=None, train: bool = False, _only=None,
                _values=None) -> list:
        """feeds: global tensors for every placeholder and parameter, or
        already-sharded lists (node id -> list of local shards).
        train=True keeps what backward() needs: every matmul's operands in
        the layouts its strategy consumed them, and every GELU's input (the
        fused GELU's epilogue then also stores its pre-activation) -- except
        for the stages the plan's checkpoint schedule recomputes, whose state
        is dropped after the pass and rebuilt by backward (_only / _values:
        that recompute: only these nodes, from these boundary values)."""
        from .runtime import gelu

        values, converted, fused = dict(_values or {}), {}, set()
        if _only is None:
            self._saved = {} if train else None
            begin = getattr(self.mesh, "begin_step", None)
            if begin is not None:  # recycle a per-step allocator (peer runtime heap)
                begin(stream)
        for n in self.graph["nodes"]:
            nid, kind = n["id"], n["kind"]
            if _only is not None and nid not in _only:
                continue
            if kind in ("placeholder", "parameter"):
                v = feeds[nid]
                values[nid] = v if isinstance(v, list) else self.shard(nid, v)
                continue
            if nid in self._attn_members and not train:
                continue  # computed inside the fused softmax below
            if nid in self._attn and not train:
                from . import block_ops as B
                _, _, _, x, m, alpha = self._attn[nid]
                outs = [self._empty(t.shape, t.dtype, t.device) for t in values[x]]
                for xs, ms, o in zip(values[x], values[m], outs):
                    B.masked_softmax(xs, o, alpha, ms, MASK_FILL, stream=stream)
                values[nid] = outs
                continue
            ins = []
            gather_b = ((kind == "matmul" and not train and self._gatherable_b(nid))
                        or (kind == "embedding-lookup" and self._gatherable_table(nid)))
            for slot, (src, _) in enumerate(n["inputs"]):
                have, want = self.spec[src], self.required_spec(nid, slot)
                if have == want or (slot == 1 and gather_b):
                    ins.append(values[src])
                    continue
                key = (src, str(want))
                if key not in converted:
                    converted[key] = self._convert(src, values[src], have, want, stream)
                ins.append(converted[key])
            if kind == "matmul":
                st = self.strategy[nid]
                out_spec = self.spec[nid]
                outs = self._alloc(nid, out_spec, ins[0][0])
                gelu_node = self._fusable_gelu(nid)
                pre = None
                if train:
                    self._saved[nid] = (ins[0], ins[1])
                    if gelu_node:  # one pass writes GELU(acc) and keeps acc for backward
                        pre = self._alloc(nid, self.spec[nid], ins[0][0])
                        self._saved[gelu_node] = pre
                if gather_b:
                    self._matmul_gathered_b(nid, ins[0], ins[1], outs, gelu_node is not None,
                                            stream)
                else:
                    self.mesh.sharded_matmul(st, self._meta(n["inputs"][0][0]),
                                             self._meta(n["inputs"][1][0]), ins[0], ins[1], outs,
                                             gelu=gelu_node is not None, b_layout="kn",
                                             stream=stream, gelu_save=pre)
                if gelu_node:
                    fused.add(gelu_node)
                values[nid] = outs
            elif kind == "elementwise-unary":
                if nid in fused:
                    values[nid] = ins[0]
                else:
                    from . import block_ops as B
                    op = self.unary_op(nid)
                    outs = [self._empty(t.shape, t.dtype, t.device) for t in ins[0]]
                    for x, y in zip(ins[0], outs):
                        if op[0] == "gelu":
                            gelu(x, y, stream=stream)
                        elif op[0] == "scale":
                            B.scale(x, y, op[1], stream=stream)
                        elif op[0] == "not":
                            B.mask_not(x, y, stream=stream)
                        else:
                            raise ValueError(f"{nid}: unknown unary op {op}")
                    if train:
                        self._saved[nid] = ins[0]  # the pre-activation
                    values[nid] = outs
            elif kind == "output":
                values[nid] = ins[0]
            elif kind == "embedding-lookup" and gather_b:
                values[nid] = self._lookup_gathered_table(nid, ins[0], ins[1], stream)
                if train:
                    self._saved[nid] = ins[0]
            elif kind in _BLOCK_KINDS:
                values[nid] = self._block_node(n, ins, stream)
                if train:  # what the node's backward reads (_block_backward)
                    if kind in ("batched-matmul", "layernorm"):
                        self._saved[nid] = ins
                    elif kind == "embedding-lookup":
                        self._saved[nid] = ins[0]
                    elif kind == "softmax":
                        self._saved[nid] = values[nid]
            else:
                raise NotImplementedError(kind)
        if _only is not None:
            return None
        if train and self._blocks:
            # checkpointed stages: keep each block's boundary inputs, drop the
            # backward state of its members (rebuilt by _recompute_block)
            self._ckpt_values = {}
            for members in self._blocks.values():
                inside = set(members)
                for m in members:
                    for src, _ in self.nodes[m]["inputs"]:
                        if src not in inside:
                            self._ckpt_values[src] = values[src]
                    self._saved.pop(m, None)
            self._recomputed = set()
        return values[self.graph["output"]]

    def _recompute_block(self, b: int, stream) -> None:
        """Re-run checkpoint block b's forward from its boundary values,
        keeping what backward needs (the schedule's second f_all pass)."""
        self.forward(None, stream=stream, train=True, _only=set(self._blocks[b]),
                     _values=self._ckpt_values)
        self._recomputed.add(b)

    def _block_node(self, n: dict, ins: list, stream) -> list:
        """One transformer-block node on every local shard (module docstring)."""
        from . import block_ops as B

        nid, kind = n["id"], n["kind"]
        spec = self.spec[nid]
        local = spec.local_shape(self._meta(nid), self.geo)
        if kind == "reshape":  # a view: the plan's rewritten local target shape
            return [x.view(local) for x in ins[0]]
        if kind == "embedding-lookup":
            outs = [self._empty(local, t.dtype, t.device) for t in ins[1]]
            for ids, table, o in zip(ins[0], ins[1], outs):
                B.embedding(ids, table, o, stream=stream)
            return outs
        dt = next(x[0].dtype for x in ins if x[0].dtype != torch.uint8)
        outs = [self._empty(local, dt, ins[0][0].device) for _ in range(self.mesh.num_local)]
        if kind == "layernorm":
            g = ins[1] if len(ins) > 1 else [None] * len(outs)
            b = ins[2] if len(ins) > 2 else [None] * len(outs)
            for x, gg, bb, o in zip(ins[0], g, b, outs):
                B.layernorm(x, gg, bb, o, stream=stream)
        elif kind == "softmax":
            axis = n.get("attrs", {}).get("axis", -1)
            for x, o in zip(ins[0], outs):
                if axis in (-1, len(local) - 1):
                    B.softmax(x, o, stream=stream)
                else:  # the strategy keeps the softmax axis whole on every device
                    B.softmax_axis(x, o, axis, stream=stream)
        elif kind == "transpose":
            perm = list(n["attrs"]["perm"])
            r = len(perm)
            for x, o in zip(ins[0], outs):
                if perm == list(range(r - 2)) + [r - 1, r - 2]:
                    B.transpose_last2(x, o, stream=stream)
                else:
                    B.permute(x, o, perm, stream=stream)
        elif kind == "elementwise-binary":
            a, b = ins
            if a[0].dtype == torch.uint8:
                a, b = b, a
            alpha = MASK_FILL if b[0].dtype == torch.uint8 else 1.0
            for x, y, o in zip(a, b, outs):
                B.add(x, y, o, alpha, stream=stream)
        elif kind == "batched-matmul":
            # one grouped tcgen05 GEMM per device: a problem per local batch
            st = self.strategy[nid]
            for a, b, o in zip(ins[0], ins[1], outs):
                B.bmm(a, b, o, stream=stream)
            if st.partial_sum:  # split-k strategies: `<host>.ar` (planner.cpp:263-282)
                self.mesh.all_reduce(list(st.reduce_axes), outs, stream=stream)
        return outs


    # ---- all-gather -> GEMM fusion -------------------------------------------
    def _gatherable_b(self, nid: str) -> bool:
        """A matmul whose weight is stored sharded and consumed replicated
        (the reference's budget plans: all-gather steps before split-m GEMMs)
        can read the weight's blocks straight from the devices that hold them
        -- on a simulated mesh from their buffers, on the peer runtime over
        peer memory -- as the K-slices of one grouped GEMM: the all-gather
        fused into the GEMM, no gathered copy."""
        fg = self.fuse_gather
        if fg is None:
            fg = hasattr(self.mesh, "gather_begin")
        if not fg:
            return False
        st = self.strategy[nid]
        b_src = self.nodes[nid]["inputs"][1][0]
        have = self.spec[b_src]
        if st.partial_sum or have == st.b or any(d.axes for d in st.b.dims):
            return False
        if len(have.dims) != 2 or not (not self.mesh.distributed or
                                       hasattr(self.mesh, "gather_begin")):
            return False
        shape = self.geo.shape
        nk = 1
        for a in have.dims[0].axes:
            nk *= shape[a]
        K = self.shapes[b_src][0][0]
        return nk <= 8 and (K // nk * 2) % 16 == 0

    def _matmul_gathered_b(self, nid, a_shards, b_shards, outs, gelu, stream):
        from .runtime import gemm_grouped

        b_src = self.nodes[nid]["inputs"][1][0]
        have = self.spec[b_src]
        shape = self.geo.shape
        ak, an = have.dims[0].axes, have.dims[1].axes
        nk = nn = 1
        for a in ak:
            nk *= shape[a]
        for a in an:
            nn *= shape[a]
        (K, N), _ = self.shapes[b_src]
        kb, nb = K // nk, N // nn

        def owner(i, j):  # a device holding block (i, j): mixed radix, first axis most significant
            coord = [0] * self.geo.rank()
            for axes, v in ((ak, i), (an, j)):
                for a in reversed(axes):
                    coord[a] = v % shape[a]
                    v //= shape[a]
            return self.geo.device_of(coord)

        peer = self.mesh.distributed
        if peer:  # publish this rank's weight block; read the owners' over peer memory
            staged = self.mesh.gather_begin(b_shards[0], stream)
            bptr = lambda d: self.mesh.peer_ptr(staged, d)  # noqa: E731
        else:
            bptr = lambda d: b_shards[d].data_ptr()  # noqa: E731
        a_ptrs, b_ptrs, c_ptrs = [], [], []
        eb = outs[0].element_size()
        for a, c in zip(a_shards, outs):
            for j in range(nn):
                for i in range(nk):
                    a_ptrs.append(a.data_ptr() + i * kb * 2)
                    b_ptrs.append(bptr(owner(i, j)))
                c_ptrs.append(c.data_ptr() + j * nb * eb)
        m = a_shards[0].numel() // K
        gemm_grouped(a_ptrs, b_ptrs, c_ptrs, nk, m, nb, kb, K, nb, N, "kn", outs[0].dtype, gelu,
                     stream)
        if peer:
            self.mesh.gather_end(stream)

    # ---- all-gather -> embedding lookup fusion -------------------------------
    def _block_owner(self, spec: ShardingSpec, index: tuple) -> int:
        """A device holding block `index` of `spec` (mixed radix over each
        dim's axes, first axis most significant -- the shard() layout)."""
        shape = self.geo.shape
        coord = [0] * self.geo.rank()
        for dim, v in zip(spec.dims, index):
            for a in reversed(dim.axes):
                coord[a] = v % shape[a]
                v //= shape[a]
        return self.geo.device_of(coord)

    def _block_index(self, dim, device: int) -> tuple:
        """(index, count) of `device`'s block along a dim sharded over dim.axes."""
        coord = self.geo.coord_of(device)
        idx, cnt = 0, 1
        for a in dim.axes:
            idx = idx * self.geo.shape[a] + coord[a]
            cnt *= self.geo.shape[a]
        return idx, cnt

    def _gatherable_table(self, nid: str) -> bool:
        """An embedding whose table is stored sharded (`src:S0R` / `S0S1`
        parameters of the reference's block plans) and consumed with more of
        it replicated: the lookup reads each id's row from the device owning
        that block -- the table's all-gather fused into the lookup, no
        gathered copy of a [vocab, hidden] table per device. On by default
        (fuse_gather=False disables it)."""
        if self.fuse_gather is False:
            return False
        if self.mesh.distributed and not hasattr(self.mesh, "gather_begin"):
            return False
        src = self.nodes[nid]["inputs"][1][0]
        have, want = self.spec[src], self.required_spec(nid, 1)
        if have == want:
            return False
        nb = 1
        for d in have.dims:
            for a in d.axes:
                nb *= self.geo.shape[a]
        return nb <= 64

    def _lookup_gathered_table(self, nid, ids, table, stream):
        from . import block_ops as B

        src = self.nodes[nid]["inputs"][1][0]
        have, want = self.spec[src], self.required_spec(nid, 1)
        (vocab, width), _ = self.shapes[src]
        nvb = self._block_index(have.dims[0], 0)[1]
        nhb = self._block_index(have.dims[1], 0)[1]
        peer = self.mesh.distributed
        if peer:  # publish this rank's block; read the owners' over peer memory
            staged = self.mesh.gather_begin(table[0], stream)
            ptr = lambda d: self.mesh.peer_ptr(staged, d)  # noqa: E731
        else:
            ptr = lambda d: table[d].data_ptr()  # noqa: E731
        blocks = [ptr(self._block_owner(have, (i, j))) for i in range(nvb) for j in range(nhb)]
        local = self.spec[nid].local_shape(self._meta(nid), self.geo)
        devs = [self.mesh.first_local] if peer else range(self.mesh.num_local)
        outs = []
        for d, x in zip(devs, ids):
            j, nw = self._block_index(want.dims[1], d)
            o = self._empty(local, table[0].dtype, table[0].device)
            B.embedding_blocks(x, blocks, nvb, nhb, vocab, width, j * (width // nw), o,
                               stream=stream)
            outs.append(o)
        if peer:
            self.mesh.gather_end(stream)
        return outs

    # ---- backward ---------------------------------------------
    def _convert_grad(self, nid, shards, have, want, stream):
        """Gradient of node `nid`'s value, held in layout `have`, into layout
        `want`. A layout conversion is the identity on the global tensor, so
        its adjoint is the identity too: the gradient takes the reverse
        conversion (the reference prices exactly this path for the backward
        pass, ckpt.cpp:348-356). Gradients here are never partial -- every
        partial sum is reduced where it is produced -- so the reverse path is
        exact."""
        if have == want:
            return shards
        shape, _ = self.shapes[nid]
        meta = TensorMeta(shape, shards[0].element_size())
        key = ("grad", nid, str(have), str(want), meta.dtype_bytes)
        conv = self._convs.get(key)
        if conv is None:
            conv = self.mesh.prepare(find_transform_path(have, want, self.geo, meta), meta,
                                     fuse=self.fuse)
            self._convs[key] = conv
        outs = [self._empty(want.local_shape(meta, self.geo), shards[0].dtype, shards[0].device)
                for _ in range(self.mesh.num_local)]
        conv(shards, outs, stream=stream)
        return outs

    def backward(self, grad_out, stream=None, input_grads: bool = False) -> dict:
        """Backward pass of the last forward(train=True).

        grad_out: gradient of the output (global tensor, or its RR shards).
        Returns {node id: gradient shards in the node's plan spec} for every
        parameter (fp32) and, with input_grads, every placeholder (bf16).

        Per matmul (reverse graph order): dA = dC . B^T and dB = A^T . dC on
        each device's shards (tcgen05, apl_sharded_matmul_backward), each
        summed over the mesh axes it is partial over -- for dB that is the
        data-parallel gradient all-reduce the reference prices over replica
        axes (ckpt.cpp:359-395, planner.cpp:358-385); on a simulated mesh the
        sum is fused into the GEMM. A GELU feeding A (in A's layout, single
        consumer) has its backward fused into the dA epilogue. Gradients then
        take the reverse conversion back to the producer's layout."""
        if self._saved is None:
            raise RuntimeError("backward() needs a preceding forward(train=True)")
        out_id = self.graph["output"]
        out_node = self.nodes[out_id]
        src = out_node["inputs"][0][0]
        rr = self.required_spec(out_id, 0)
        if isinstance(grad_out, list):
            g = grad_out
        else:
            g = [grad_out.to(torch.bfloat16).contiguous() for _ in range(self.mesh.num_local)]
        grads = {src: self._convert_grad(src, g, rr, self.spec[src], stream)}
        done = set()
        kinds = {"parameter"} | ({"placeholder"} if input_grads else set())

        from . import block_ops as B

        def add(nid, shards):
            if nid in grads:  # a value with several consumers: sum their gradients
                # (out of place: a gradient list may be shared with another
                # node's, e.g. both operands of a residual add)
                summed = []
                for acc, x in zip(grads[nid], shards):
                    if acc.dtype != x.dtype:
                        raise TypeError(f"{nid}: gradient dtypes differ")
                    o = self._empty(acc.shape, acc.dtype, acc.device)
                    B.add(acc, x, o, stream=stream)
                    summed.append(o)
                grads[nid] = summed
            else:
                grads[nid] = shards

        def wants_grad(nid):
            k = self.nodes[nid]["kind"]
            return k not in ("placeholder", "parameter") or k in kinds

        def ensure(nid):  # a checkpointed node's backward state, recomputed on demand
            b = self._block_of.get(nid)
            if b is not None and b not in self._recomputed:
                self._recompute_block(b, stream)

        for n in reversed(self.graph["nodes"]):
            nid, kind = n["id"], n["kind"]
            if nid in done or nid not in grads:
                continue
            dy = grads[nid]
            ensure(nid)
            if kind == "matmul":
                st = self.strategy[nid]
                a_saved, b_saved = self._saved[nid]
                a_src, b_src = n["inputs"][0][0], n["inputs"][1][0]
                ensure(a_src)  # a GELU feeding A: its saved input decides the fusion
                a_meta, b_meta = self._meta(a_src), self._meta(b_src)
                # GELU producing A in A's layout: its backward rides the dA epilogue.
                aux, a_target = None, a_src
                an = self.nodes[a_src]
                if (an["kind"] == "elementwise-unary" and self.unary_op(a_src) == ("gelu",)
                        and self.spec[a_src] == st.a
                        and len(self._consumers.get(a_src, [])) == 1
                        and isinstance(self._saved.get(a_src), list)):
                    aux, a_target = self._saved[a_src], an["inputs"][0][0]
                    done.add(a_src)
                need_a = wants_grad(a_target)
                need_b = wants_grad(b_src)
                ga = [self._empty(t.shape, t.dtype, t.device) for t in a_saved] if need_a else None
                gb = [self._empty(t.shape, torch.float32, t.device)
                      for t in b_saved] if need_b else None
                if need_a or need_b:
                    self.mesh.sharded_matmul_backward(st, a_meta, b_meta, a_saved, b_saved, dy,
                                                      ga, gb, b_layout="kn", gelu_aux=aux,
                                                      stream=stream)
                if need_a:
                    add(a_target, self._convert_grad(a_target, ga, st.a, self.spec[a_target],
                                                      stream))
                if need_b:
                    add(b_src, self._convert_grad(b_src, gb, st.b, self.spec[b_src], stream))
            elif kind == "elementwise-unary" and self.unary_op(nid)[0] == "gelu":
                from .runtime import gelu_backward
                x_src = n["inputs"][0][0]
                pre = self._saved[nid]
                dx = [self._empty(t.shape, t.dtype, t.device) for t in pre]
                for a, x, o in zip(dy, pre, dx):
                    gelu_backward(a, x, o, stream=stream)
                add(x_src, self._convert_grad(x_src, dx, self.spec[nid], self.spec[x_src], stream))
            elif kind in _BLOCK_KINDS or kind == "elementwise-unary":
                for slot, g, *lay in self._block_backward(n, dy, wants_grad, stream):
                    src = n["inputs"][slot][0]
                    have = lay[0] if lay else self.required_spec(nid, slot)
                    add(src, self._convert_grad(src, g, have, self.spec[src], stream))
        return {nid: grads[nid] for nid in grads
                if self.nodes[nid]["kind"] in kinds}


    def _block_backward(self, n: dict, dy: list, wants_grad, stream) -> list:
        """Input gradients of one block node, each in the layout the node
        consumed that input in (its strategy's input spec): [(slot, shards)].
        Gradients that are partial sums over mesh axes (parameters shared by
        sharded rows, batched-matmul contractions over a sharded dim) are
        all-reduced here, before any reverse conversion (§4.4's rule)."""
        from . import block_ops as B

        nid, kind = n["id"], n["kind"]
        ins = [i[0] for i in n["inputs"]]
        like = lambda ts, dt=None: [self._empty(t.shape, dt or t.dtype, t.device)  # noqa: E731
                                    for t in ts]
        out = []
        if kind == "reshape":
            shape = self.required_spec(nid, 0).local_shape(self._meta(ins[0]), self.geo)
            out.append((0, [g.view(shape) for g in dy]))
        elif kind == "transpose":
            perm = list(n["attrs"]["perm"])
            r = len(perm)
            inv = [perm.index(d) for d in range(r)]  # dx = dy permuted back
            dx = [self._empty(tuple(g.shape[i] for i in inv), g.dtype, g.device) for g in dy]
            for g, o in zip(dy, dx):
                if perm == list(range(r - 2)) + [r - 1, r - 2]:
                    B.transpose_last2(g, o, stream=stream)
                else:
                    B.permute(g, o, inv, stream=stream)
            out.append((0, dx))
        elif kind == "elementwise-unary":
            op = self.unary_op(nid)
            if op[0] == "scale" and wants_grad(ins[0]):
                dx = like(dy)
                for g, o in zip(dy, dx):
                    B.scale(g, o, op[1], stream=stream)
                out.append((0, dx))
            elif op[0] != "not":
                raise NotImplementedError(f"backward of unary {op}")
        elif kind == "elementwise-binary":
            for slot, src in enumerate(ins):
                if self.shapes[src][1] != 1 and wants_grad(src):  # u8 masks carry no gradient
                    out.append((slot, dy))
        elif kind == "softmax":
            y = self._saved[nid]
            dx = like(dy)
            axis = n.get("attrs", {}).get("axis", -1)
            for yy, g, o in zip(y, dy, dx):
                if axis in (-1, yy.dim() - 1):
                    B.softmax_backward(yy, g, o, stream=stream)
                else:
                    B.softmax_axis_backward(yy, g, o, axis, stream=stream)
            out.append((0, dx))
        elif kind == "layernorm":
            x, *aff = self._saved[nid]
            gamma = aff[0] if aff else [None] * len(x)
            dx = like(dy)
            h = x[0].shape[-1]
            dg = [self._zeros((h,), t.device) for t in x] if aff else None
            db = [self._zeros((h,), t.device) for t in x] if len(aff) > 1 else None
            for i, (xx, gg, g, o) in enumerate(zip(x, gamma, dy, dx)):
                B.layernorm_backward(xx, gg, g, o, dg[i] if dg else None, db[i] if db else None,
                                     stream=stream)
            out.append((0, dx))
            # gamma / beta are replicated; each device summed its own rows
            row_axes = sorted({a for d in self.required_spec(nid, 0).dims[:-1] for a in d.axes})
            for slot, pg in ((1, dg), (2, db)):
                if pg is not None and wants_grad(ins[slot]):
                    if row_axes:
                        self.mesh.all_reduce(row_axes, pg, stream=stream)
                    out.append((slot, pg))
        elif kind == "embedding-lookup":
            ids = self._saved[nid]
            tspec, tplan = self.required_spec(nid, 1), self.spec[ins[1]]
            if (wants_grad(ins[1]) and not self.mesh.distributed and not tspec.dims[1].axes
                    and tplan != tspec):
                # straight into the table's own layout: reduce-scatter fused
                out.append((1, self._embedding_grad_owned(nid, ids, dy, tplan, stream), tplan))
            elif wants_grad(ins[1]):
                shape = tspec.local_shape(self._meta(ins[1]), self.geo)
                dt = [self._zeros(shape, g.device) for g in dy]
                for i, g, o in zip(ids, dy, dt):
                    B.embedding_backward(i, g, o, stream=stream)
                id_axes = sorted({a for d in self.required_spec(nid, 0).dims for a in d.axes})
                if id_axes:  # replicated table rows, ids sharded: partial sums
                    self.mesh.all_reduce(id_axes, dt, stream=stream)
                out.append((1, dt))
        elif kind == "batched-matmul":
            st = self.strategy[nid]
            a, b = self._saved[nid]
            # dA = dC . B^T partial over the axes sharding C's n dim, dB = A^T . dC
            # over those sharding C's m dim (each device holds whole batches).
            # Split-k strategies (partial_sum, intraop.cpp:208-231): the forward
            # all-reduce over reduce_axes hands every partial the whole dC, so
            # each device's k-shard gradients are dC . B_k^T and A_k^T . dC --
            # the same local products, no extra reduction over reduce_axes.
            if wants_grad(ins[0]):
                da = like(a)
                for g, bb, o in zip(dy, b, da):
                    B.bmm(g, bb, o, b_t=True, stream=stream)
                if st.c.dims[2].axes:
                    self.mesh.all_reduce(list(st.c.dims[2].axes), da, stream=stream)
                out.append((0, da))
            if wants_grad(ins[1]):
                db = like(b)
                for aa, g, o in zip(a, dy, db):
                    B.bmm(aa, g, o, a_t=True, stream=stream)
                if st.c.dims[1].axes:
                    self.mesh.all_reduce(list(st.c.dims[1].axes), db, stream=stream)
                out.append((1, db))
        else:
            raise NotImplementedError(f"backward through {kind} ({nid})")
        return out

    def _embedding_grad_owned(self, nid, ids, dy, tplan, stream) -> list:
        """Table gradient of an embedding whose table is consumed with the
        hidden dim whole (emb-batch) but stored sharded (`tplan`): every
        device accumulates only its own block, from one representative
        source per distinct id block (replicas counted once). Replaces a
        [vocab, width] fp32 partial per device + all-reduce + slice."""
        from . import block_ops as B

        ispec = self.required_spec(nid, 0)
        srcs = {}
        for d in range(self.mesh.num_local):
            key = tuple(self._block_index(dim, d)[0] for dim in ispec.dims)
            srcs.setdefault(key, d)
        order = sorted(srcs.values())
        src_ids = [ids[d] for d in order]
        src_dy = [dy[d] for d in order]
        (vocab, width), _ = self.shapes[self.nodes[nid]["inputs"][1][0]]
        outs = []
        for d in range(self.mesh.num_local):
            iv, nv = self._block_index(tplan.dims[0], d)
            ih, nh = self._block_index(tplan.dims[1], d)
            blk = self._zeros((vocab // nv, width // nh), dy[0].device)
            B.embedding_backward_block(src_ids, src_dy, blk, iv * (vocab // nv),
                                       ih * (width // nh), stream=stream)
            outs.append(blk)
        return outs

    # ---- CUDA graphs ---------------------------------------------------------
    def capture(self, feeds: dict, grad_out=None, warmup: int = 1):
        """Record one step -- forward, or forward + backward when grad_out is
        given -- into a CUDA graph and return (replay, outputs, grads): every
        launch of the step (conversion kernels, GEMMs, all-reduces) replays
        with no host work. The outputs / grads are the graph's own buffers,
        rewritten by each replay; feeds must stay at the same addresses (copy
        new data into them between replays)."""
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        train = grad_out is not None
        with torch.cuda.stream(side):
            for _ in range(max(1, warmup)):  # compiles every exchange / tensor map
                self.forward(feeds, stream=side, train=train)
                if train:
                    self.backward(grad_out, stream=side)
            side.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=side):
                outs = self.forward(feeds, stream=side, train=train)
                grads = self.backward(grad_out, stream=side) if train else None
        torch.cuda.current_stream().wait_stream(side)
        return graph.replay, outs, grads


def megatron_mlp_plan(mesh_rank: int = 1, axis: int = 0) -> dict:
    """BASELINE config 5 pinned selection on a mesh axis: fc1 split-n (RR x RS
    -> RS, GELU fused), fc2 split-k (RS x SR -> RR partial, all-reduce).
    Same document shape as plan_to_json (nodes + inserted_comm_nodes)."""
    r = "R" * 1
    s = f"S{axis}"
    rr = "RR" if mesh_rank >= 1 else r
    nodes = {
        "x": {"strategy": f"src:{rr}", "spec": rr, "partial_sum": False},
        "w1": {"strategy": f"src:R{s}", "spec": f"R{s}", "partial_sum": False},
        "w2": {"strategy": f"src:{s}R", "spec": f"{s}R", "partial_sum": False},
        "fc1": {"strategy": f"split-n:{axis}", "spec": f"R{s}", "partial_sum": False},
        "gelu": {"strategy": f"split-n:{axis}", "spec": f"R{s}", "partial_sum": False},
        "fc2": {"strategy": f"split-k:{axis}", "spec": rr, "partial_sum": True,
                "reduce_axes": [axis]},
        "out": {"strategy": "collect", "spec": rr, "partial_sum": False},
    }
    return {"version": 1, "nodes": nodes,
            "inserted_comm_nodes": [{"node": "fc2.ar", "producer": "fc2", "producer_out": 0,
                                     "collective": "all-reduce", "axes": [axis], "bytes": 0}]}

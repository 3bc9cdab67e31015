"""ComputationGraph of the drop-in API (pkg/src/dyncore/graph.py:20-172).

Construction stays on the host and keeps the reference contract: add_node
checks staleness and runs the shape rule immediately (errors at construction,
no numeric work), nodes are append-only, `renew()` bumps the generation.
Execution is delegated in bulk to the native executor (libdyngpu.so): the
pending node records are packed into one dg_node table per call
(dg_graph_append), `forward_to`/`value` evaluate only nodes past the
watermark (incremental, never recomputes), `backward` runs the batched
reverse sweep with gradients landing in the Model's device storage.

Counters keep the reference's semantics: `forward_calls` counts nodes
(including parameter aliases), the pools' alloc_count/cursor charge the same
64-byte-rounded sizes per node (arena.py:48-56).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _dgcore, _native
from . import device as _dev
from .errors import NonScalarLoss, ShapeError, StaleExpression
from .ops import FAST_KINDS, REGISTRY
from .params import materialize_pending
from .tensor import Shape, Tensor


class Expression(_dgcore.ExprBase):
    """Handle to a graph node; valid for one graph generation (storage in the
    _dgcore base type; instances are created by the native add_node)."""

    __slots__ = ()

    def __init__(self, graph: "ComputationGraph", index: int, generation: int):
        self.graph = graph
        self.index = index
        self.generation = generation

    @property
    def shape(self) -> Shape:
        self.graph.check_current(self)
        return self.graph.nodes[self.index].shape

    def __repr__(self) -> str:
        return f"Expression(node={self.index}, gen={self.generation})"


class Node(_dgcore.NodeBase):
    __slots__ = ()

    def __init__(self, kind: str, inputs: tuple, shape: Shape, aux, code: int):
        self.kind = kind
        self.inputs = inputs
        self.shape = shape
        self.aux = aux
        self.code = code


class ModelGradientSink:
    """Default backward target: the parameters' own gradient storage
    (graph.py:51-66).  The device executor accumulates into it directly.  Any
    other object assigned to `cg.sink` receives the reference sink protocol
    (`add_param_grad`, `add_lookup_rows_grad`) after the device backward, see
    ComputationGraph._backward_to_sink."""

    def add_param_grad(self, p, flat) -> None:
        g = p.gradient.data
        g += np.asarray(flat, dtype=g.dtype).reshape(g.shape)

    def add_lookup_row_grad(self, lp, row: int, vec) -> None:
        self.add_lookup_rows_grad(lp, [row], np.asarray(vec).reshape(1, -1))

    def add_lookup_rows_grad(self, lp, ids, rows) -> None:
        g = lp.gradient
        np.add.at(g, list(ids), np.asarray(rows, dtype=g.dtype).reshape(len(ids), -1))
        lp.touched = lp.touched | set(int(i) for i in ids)


DIRECT_SINK = ModelGradientSink()

_HDR_FIELDS = 13


class ComputationGraph:
    def __init__(self, pools):
        self.pools = pools
        self.dtype = pools.dtype
        self.nodes: list[Node] = []
        self.generation = 0
        self.watermark = -1
        self.forward_calls = 0
        self.sink = DIRECT_SINK
        self._h = None  # native dg_graph*
        self._sent = 0  # nodes already appended to the native table
        # native construction (csrc/dgcore.c): node records are encoded as the
        # graph is built; add_node is the C fast path bound per instance
        self._core = _dgcore.GraphCore(self, self.nodes)
        self.add_node = self._core.add
        self._stream = None
        pools.bind(self)

    # -- native plumbing ---------------------------------------------------

    def _native(self):
        if self._h is None:
            lib = _native.lib()
            fwd, bwd, work = self.pools.device_buffers()
            h = ctypes.c_void_p()
            _native.check(lib.dg_graph_create(
                _dev.torch().cuda.current_device(), _native.ptr(fwd), self.pools.forward.capacity,
                _native.ptr(bwd), self.pools.backward.capacity, _native.ptr(work), self.pools.work_bytes,
                ctypes.byref(h)))
            self._h = h
        s = _dev.stream_ptr()
        if s != self._stream:
            _native.check(_native.lib().dg_graph_set_stream(self._h, s))
            self._stream = s
        return self._h

    def _counters(self):
        out = np.zeros(8, dtype=np.int64)
        if self._h is not None:
            _native.check(_native.lib().dg_graph_counters(self._h, out.ctypes.data))
        return out

    def plan_stats(self):
        out = np.zeros(8, dtype=np.int64)
        if self._h is not None:
            _native.check(_native.lib().dg_graph_plan_stats(self._h, out.ctypes.data))
        return out

    def profile_enable(self, classes) -> None:
        """CUDA-event timing of every launch of the given op classes
        (names from _native.PROFILE_CLASSES)."""
        mask = 0
        for c in classes:
            mask |= 1 << _native.PROFILE_CLASSES.index(c)
        _native.check(_native.lib().dg_profile_enable(self._native(), mask))

    def profile_read(self, cls: str) -> dict:
        out = np.zeros(4, dtype=np.float64)
        _native.check(_native.lib().dg_profile_read(self._native(), _native.PROFILE_CLASSES.index(cls),
                                                    out.ctypes.data))
        return {"ms": float(out[0]), "launches": int(out[1]), "flops": float(out[2]), "bytes": float(out[3])}

    def profile_reset(self) -> None:
        _native.check(_native.lib().dg_profile_reset(self._native()))

    def _native_renew(self):
        if self._h is not None:
            _native.check(_native.lib().dg_graph_renew(self._h))

    def __del__(self):
        try:
            if self._h is not None:
                _native.lib().dg_graph_destroy(self._h)
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    def _flush(self, h) -> None:
        """Hand the pending node records (encoded at construction by the
        native add_node) to the executor as one dg_node table."""
        start, end = self._sent, len(self.nodes)
        if start == end:
            return
        hdr, n, ins, n_ins, ai, n_ai, af, n_af = self._core.pack(start)
        _native.check(_native.lib().dg_graph_append(h, hdr, n, ins, n_ins, ai, n_ai, af, n_af))
        self._sent = end

    def _prepare(self):
        materialize_pending()
        h = self._native()
        self._flush(h)
        return h

    # -- lifecycle ---------------------------------------------------------

    def renew(self) -> None:
        self.nodes.clear()
        self.generation += 1
        self.watermark = -1
        self._sent = 0
        self._core.renew(self.generation)
        self.pools.reset_transient()

    def check_current(self, e: Expression) -> None:
        if e.graph is not self or e.generation != self.generation:
            raise StaleExpression(
                f"expression from generation {e.generation} used in generation {self.generation}"
            )

    # -- construction ------------------------------------------------------

    def add_node(self, kind: str, inputs=(), aux=None) -> Expression:  # noqa: F811 - per-instance native override
        """Reference-semantics add_node (graph.py:97-106); instances use the
        native GraphCore.add bound in __init__, which runs the same checks and
        shape rules (deferring to the Python rules for anything irregular)."""
        return self._core.add(kind, tuple(inputs), aux)

    def _add_node_py(self, kind: str, inputs=(), aux=None) -> Expression:
        gen = self.generation
        nodes = self.nodes
        in_shapes = []
        indices = []
        for e in inputs:
            if e.graph is not self or e.generation != gen:
                self.check_current(e)
            in_shapes.append(nodes[e.index].shape)
            indices.append(e.index)
        od = REGISTRY[kind]
        shape = od.shape(aux, in_shapes)
        nodes.append(Node(kind, tuple(indices), shape, aux, od.code))
        return Expression(self, len(nodes) - 1, gen)

    # -- evaluation --------------------------------------------------------

    def _advance(self, upto: int) -> None:
        if upto > self.watermark:
            self.forward_calls += upto - self.watermark
            self.watermark = upto

    def forward_to(self, e: Expression) -> None:
        self.check_current(e)
        if e.index <= self.watermark:
            return
        h = self._prepare()
        _native.check(_native.lib().dg_forward(h, e.index))
        self._advance(e.index)

    def value(self, e: Expression) -> Tensor:
        """Host copy of a node value (graph.py:132-135); synchronises."""
        self.check_current(e)
        h = self._prepare()
        shape = self.nodes[e.index].shape
        out = np.empty(shape.size(), dtype=np.float32)
        _native.check(_native.lib().dg_value(h, e.index, out.ctypes.data, out.shape[0]))
        self._advance(e.index)
        return Tensor(shape, out)

    # -- differentiation ---------------------------------------------------

    def backward(self, e: Expression) -> None:
        self.check_current(e)
        loss = self.nodes[e.index]
        if loss.shape.elem_size() != 1 or loss.shape.batch != 1:
            raise NonScalarLoss(f"backward needs a scalar, got {loss.shape}")
        if self.sink is not DIRECT_SINK:
            self._backward_to_sink(e)
            return
        h = self._prepare()
        _native.check(_native.lib().dg_backward(h, e.index))
        self._advance(e.index)
        _dev.bump_epoch()

    def _backward_to_sink(self, e: Expression) -> None:
        """backward() with a custom sink (graph.py:139-164 flushing through
        `self.sink`, e.g. the reference's GradientSlots, parallel.py:30-46).

        The device backward runs unchanged into zeroed gradient storage of
        every parameter / lookup table a node <= loss references (all nodes
        <= loss flush, ancestors or not); the result is handed to the sink as
        ONE `add_param_grad(p, flat)` per parameter and ONE
        `add_lookup_rows_grad(lp, ids, rows)` per table with the sorted unique
        rows this backward touched, then the model's own gradients and touched
        sets are restored.  For an additive sink this equals the reference's
        per-node flushes up to the order of fp32 additions."""
        h = self._prepare()
        params, tables, seen = [], [], set()
        for node in self.nodes[: e.index + 1]:
            if node.kind == "parameter":
                x = node.aux
            elif node.kind in ("lookup", "lookup_batch"):
                x = node.aux[0]
            else:
                continue
            if id(x) in seen:
                continue
            seen.add(id(x))
            (params if node.kind == "parameter" else tables).append(x)
        saved = []
        for x in params + tables:
            saved.append(x._gm.dev.clone())
            x._gm.dev.zero_()
        touched = [lp.touched for lp in tables]
        for lp in tables:
            lp.touched = ()
        _native.check(_native.lib().dg_backward(h, e.index))
        self._advance(e.index)
        grads = []
        for x, keep in zip(params + tables, saved):
            if x in tables:
                ids = np.array(sorted(x.touched), dtype=np.int64)
                it = _dev.torch().from_numpy(ids).to(x._gm.dev.device)
                rows = x._gm.dev.view(x.rows, x.dim).index_select(0, it).cpu().numpy()
                grads.append((ids, rows))
            else:
                grads.append(x._gm.dev.cpu().numpy())
            x._gm.dev.copy_(keep)
        for lp, t in zip(tables, touched):
            lp.touched = t
        _dev.bump_epoch()
        for x, g in zip(params + tables, grads):
            if x in tables:
                self.sink.add_lookup_rows_grad(x, [int(i) for i in g[0]], g[1])
            else:
                self.sink.add_param_grad(x, g)

    def gradient(self, e: Expression) -> Tensor:
        """Debug accessor for a node's last backward slot.  Parameter nodes
        accumulate straight into the parameter gradient, so for them this is
        the parameter's accumulated gradient."""
        self.check_current(e)
        shape = self.nodes[e.index].shape
        if self._h is None:
            raise ShapeError("no backward pass has populated this node yet")
        out = np.empty(shape.size(), dtype=np.float32)
        _native.check(_native.lib().dg_gradient(self._h, e.index, out.ctypes.data, out.shape[0]))
        return Tensor(shape, out)


_dgcore.setup(Shape, Node, Expression, REGISTRY, FAST_KINDS)

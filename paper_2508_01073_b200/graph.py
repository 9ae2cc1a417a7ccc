"""Device-resident CSR graph (drop-in for walkvec.graph.Graph / build_graph).

Reference: pkg/src/walkvec/graph.py:31-98.  The adjacency of vertex v is the
input-order slice of its out-edges (stable by source, graph.py:89).  On the
device the two column arrays are packed into one 8-byte word per edge,
``pred << 32 | dst``, so a walk hop reads one 8-byte edge after the two row
offsets.  ``row_offsets`` / ``col_targets`` / ``col_predicates`` are exposed
as int64 numpy arrays (materialised lazily) so reference code keeps working.
"""

from __future__ import annotations

import numpy as np

from . import _lib


class Graph:
    """Immutable directed labeled multigraph over integer tokens (device CSR)."""

    def __init__(self, vertex_count: int, d_row_offsets, d_edges, edge_count: int):
        self.vertex_count = int(vertex_count)
        self.edge_count = int(edge_count)
        self.d_row_offsets = d_row_offsets  # torch int64 [V+1] (cuda)
        self.d_edges = d_edges  # torch int64 [E] holding u64 (pred << 32 | dst)
        self._np = {}
        self._adj = None

    def walk_adjacency(self):
        """Device [E, 4] int32 {pred, dst, row start of dst, out-degree of dst} (built once, cached):
        a walk hop reads one 16-byte entry instead of offsets then edge.  None when E >= 2^32
        or WV_NO_WALK_ADJ is set (the walks then read the CSR directly)."""
        import os

        if self._adj is None:
            if self.edge_count == 0 or self.edge_count >= (1 << 32) or self.vertex_count >= (1 << 32) or \
                    os.environ.get("WV_NO_WALK_ADJ"):
                return None
            torch = _lib.require_cuda()
            adj = torch.empty((self.edge_count, 4), dtype=torch.int32, device=self.d_edges.device)
            _lib.call("wv_walk_adjacency_build", _lib.ptr(self.d_row_offsets), _lib.ptr(self.d_edges),
                      self.vertex_count, self.edge_count, _lib.ptr(adj), _lib.stream_ptr())
            self._adj = adj
        return self._adj

    # -- reference-compatible views -------------------------------------
    def _unpacked(self):
        if "targets" not in self._np:
            torch = _lib.require_cuda()
            E = self.edge_count
            t = torch.empty(max(E, 1), dtype=torch.int64, device=self.d_edges.device)
            p = torch.empty(max(E, 1), dtype=torch.int64, device=self.d_edges.device)
            if E:
                _lib.call("wv_csr_unpack", _lib.ptr(self.d_edges), E, _lib.ptr(t), _lib.ptr(p), _lib.stream_ptr())
            self._np["targets"] = t[:E].cpu().numpy()
            self._np["preds"] = p[:E].cpu().numpy()
        return self._np["targets"], self._np["preds"]

    @property
    def row_offsets(self) -> np.ndarray:
        if "offsets" not in self._np:
            self._np["offsets"] = self.d_row_offsets.cpu().numpy()
        return self._np["offsets"]

    @property
    def col_targets(self) -> np.ndarray:
        return self._unpacked()[0]

    @property
    def col_predicates(self) -> np.ndarray:
        return self._unpacked()[1]

    def out_degree(self, v: int) -> int:
        self._check_vertex(v)
        return int(self.row_offsets[v + 1] - self.row_offsets[v])

    def out_neighbors(self, v: int):
        self._check_vertex(v)
        lo, hi = self.row_offsets[v], self.row_offsets[v + 1]
        return self.col_predicates[lo:hi], self.col_targets[lo:hi]

    def edge_array(self) -> np.ndarray:
        src = np.repeat(np.arange(self.vertex_count, dtype=np.int64), np.diff(self.row_offsets))
        return np.column_stack([src, self.col_predicates, self.col_targets])

    def participating_vertices(self) -> np.ndarray:
        sources = np.flatnonzero(np.diff(self.row_offsets) > 0)
        return np.union1d(sources, np.unique(self.col_targets))

    def _check_vertex(self, v: int):
        if not 0 <= v < self.vertex_count:
            raise IndexError(f"vertex {v} out of range [0, {self.vertex_count})")

    @property
    def device(self):
        return self.d_row_offsets.device

    # -- adapters ---------------------------------------------------------
    @classmethod
    def from_csr(cls, row_offsets, col_targets, col_predicates, vertex_count=None, device=None) -> "Graph":
        """Wrap an existing host CSR (e.g. a reference walkvec Graph) on the device."""
        torch = _lib.require_cuda()
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        off = torch.as_tensor(np.asarray(row_offsets, dtype=np.int64)).to(dev)
        tg = np.asarray(col_targets, dtype=np.int64)
        pr = np.asarray(col_predicates, dtype=np.int64)
        packed = (pr << 32) | (tg & 0xFFFFFFFF)
        V = int(vertex_count) if vertex_count is not None else len(row_offsets) - 1
        g = cls(V, off, torch.as_tensor(packed).to(dev), len(tg))
        return g


def as_device_graph(graph, device=None) -> Graph:
    """Accept our Graph or any object with the reference CSR attributes."""
    if isinstance(graph, Graph):
        return graph
    cached = getattr(graph, "_b200_device_graph", None)
    if cached is not None:
        return cached
    g = Graph.from_csr(graph.row_offsets, graph.col_targets, graph.col_predicates, graph.vertex_count, device)
    try:
        object.__setattr__(graph, "_b200_device_graph", g)
    except (AttributeError, TypeError):
        pass  # __slots__ class (the reference Graph): no caching
    return g


def build_graph(edges, vertex_count: int, device=None) -> Graph:
    """Assemble a device CSR from ``(E, 3)`` token rows (graph.py:74-98).

    ``edges`` may be a numpy array / nested list or a torch tensor (host or
    device).  Errors mirror the reference: ValueError for a bad shape or a
    token outside ``[0, vertex_count)``.
    """
    torch = _lib.require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if isinstance(edges, torch.Tensor):
        e = edges.to(device=dev, dtype=torch.int64)
    else:
        arr = np.asarray(edges, dtype=np.int64)
        if arr.size == 0:
            arr = arr.reshape(0, 3)
        if arr.ndim != 2 or arr.shape[1] != 3:
            raise ValueError("edges must be an (E, 3) array")
        e = torch.from_numpy(np.ascontiguousarray(arr)).to(dev, non_blocking=False)
    if e.numel() == 0:
        e = e.reshape(0, 3)
    if e.dim() != 2 or e.shape[1] != 3:
        raise ValueError("edges must be an (E, 3) array")
    e = e.contiguous()
    E = int(e.shape[0])
    V = int(vertex_count)
    if E:
        lo, hi = torch.aminmax(e)
        if int(lo) < 0 or int(hi) >= V:
            raise ValueError("edge token out of range for vertex_count")
    if V < 1:
        raise ValueError("vertex_count must be >= 1")
    off = torch.empty(V + 1, dtype=torch.int64, device=dev)
    packed = torch.empty(max(E, 1), dtype=torch.int64, device=dev)
    ws = torch.empty(_lib.query("wv_csr_workspace_bytes", E, V), dtype=torch.uint8, device=dev)
    _lib.call("wv_csr_build", _lib.ptr(e), E, V, _lib.ptr(off), _lib.ptr(packed), _lib.ptr(ws), ws.numel(),
              _lib.stream_ptr())
    return Graph(V, off, packed[:E], E)

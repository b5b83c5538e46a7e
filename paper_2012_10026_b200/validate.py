"""BFS-tree validation on the device (reference validate.py:1-235).

Same five rules, names, report texts and ``derived_levels`` as the
reference's :class:`Validator`; the checks run in ``csrc/rb_validate.cu``
(union-find component labels, per-vertex rule kernels, pointer-jumping level
derivation, per-edge level-span check), so trees can be validated at sizes
where the reference's int64 edge keys do not fit in host memory.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .graph import CsrGraph, EdgeList, _edges_device

__all__ = ["CheckResult", "ValidationReport", "Validator", "validate"]

CHECK_NAMES = (
    "source is own parent",
    "tree edges exist",
    "parent chains are proper levels",
    "edges span at most one level",
    "reachability matches components",
)


@dataclass
class CheckResult:
    name: str
    passed: bool
    detail: str = ""


@dataclass
class ValidationReport:
    """Outcome of all five rules plus the levels derived from the tree (validate.py:38-60)."""

    passed: bool
    checks: list[CheckResult] = field(default_factory=list)
    derived_levels: np.ndarray | None = None

    def as_text(self) -> str:
        lines = [f"validation: {'PASS' if self.passed else 'FAIL'}"]
        for c in self.checks:
            status = "ok" if c.passed else "FAIL"
            suffix = f" ({c.detail})" if c.detail and not c.passed else ""
            lines.append(f"  [{status}] {c.name}{suffix}")
        return "\n".join(lines)

    def as_key_values(self) -> str:
        lines = [f"passed = {str(self.passed).lower()}"]
        for c in self.checks:
            key = c.name.replace(" ", "_")
            lines.append(f"check.{key} = {str(c.passed).lower()}")
            if c.detail and not c.passed:
                lines.append(f"check.{key}.detail = {c.detail}")
        return "\n".join(lines)


class Validator:
    """Reusable checker (validate.py:96-225): component labels computed once
    on the device, from the raw edge list when given (independent of the CSR
    build), else from the CSR."""

    def __init__(self, g: CsrGraph, edge_list: EdgeList | None = None):
        torch = _lib.require_cuda()
        self.torch = torch
        self.g = g
        L = _lib.lib()
        n = g.n
        rs, col, _ = g.device_arrays()
        self._labels = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")[:n]
        s = _lib.stream_ptr()
        if n:
            if edge_list is not None:
                ed, _ = _edges_device(edge_list)
                _lib.check(L.rb_components(None, None, n, _lib.ptr(ed), int(ed.shape[0]), _lib.ptr(self._labels), s),
                           "rb_components")
            else:
                _lib.check(L.rb_components(_lib.ptr(rs), _lib.ptr(col), n, None, 0, _lib.ptr(self._labels), s),
                           "rb_components")
        self._ws = None

    def component_labels(self) -> np.ndarray:
        """int64 labels, each the min vertex id of its component (validate.py:63-84)."""
        return self._labels.cpu().numpy().astype(np.int64)

    def component_labels_device(self):
        return self._labels

    def validate_device(self, source: int, parent):
        """Run the five rules on a device (or host) int32 predecessor array.
        Returns (first_bad[5] int64 numpy, derived levels int32 CUDA tensor,
        parent as a CUDA tensor)."""
        torch = self.torch
        g = self.g
        n = g.n
        if isinstance(parent, torch.Tensor):
            if tuple(parent.shape) != (n,):
                raise ValueError(f"predecessor array has shape {tuple(parent.shape)}, expected ({n},)")
            pd = parent.to(device="cuda", dtype=torch.int32).contiguous()
        else:
            p = np.asarray(parent)
            if p.shape != (n,):
                raise ValueError(f"predecessor array has shape {p.shape}, expected ({n},)")
            p64 = p.astype(np.int64)
            # values outside int32 are out of range parents (rule 2) -- clamp to n
            p32 = np.where(p64 >= n, n, np.where(p64 < -1, -1, p64)).astype(np.int32) if n else p64.astype(np.int32)
            pd = torch.from_numpy(np.ascontiguousarray(p32)).cuda()
        if not 0 <= source < n:
            raise ValueError(f"source {source} out of range for n={n}")
        L = _lib.lib()
        wsb = L.rb_validate_workspace_bytes(n)
        if self._ws is None or self._ws.numel() < wsb:
            self._ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        rs, col, _ = g.device_arrays()
        levels = torch.empty(n, dtype=torch.int32, device="cuda")
        bad = np.full(5, -1, np.int64)
        _lib.check(
            L.rb_validate(_lib.ptr(rs), _lib.ptr(col), n, _lib.ptr(self._labels), int(source), _lib.ptr(pd),
                          _lib.ptr(self._ws), wsb, _lib.ptr(levels), bad.ctypes.data_as(ctypes.c_void_p),
                          _lib.stream_ptr()),
            "rb_validate",
        )
        return bad, levels, pd

    def validate(self, source: int, parent) -> ValidationReport:
        bad, levels_d, pd = self.validate_device(source, parent)
        levels = levels_d.cpu().numpy().astype(np.int64)
        host_parent = None if isinstance(parent, self.torch.Tensor) else np.asarray(parent)

        def par(v):
            return int(host_parent[v]) if host_parent is not None else int(pd[v].item())

        details = ["", "", "", "", ""]
        if bad[0] >= 0:
            details[0] = f"parent[{source}] = {par(source)}"
        if bad[1] >= 0:
            v = int(bad[1])
            details[1] = f"(v={v}, parent={par(v)}) is not a graph edge"
        if bad[2] >= 0:
            details[2] = f"vertex {int(bad[2])}: parent chain never reaches the source (cycle or unreached parent)"
        if bad[3] >= 0:
            j = int(bad[3])
            rs = self.g.device_arrays()[0]
            u = int(self.torch.searchsorted(rs, self.torch.tensor([j], dtype=rs.dtype, device=rs.device),
                                            right=True).item()) - 1
            w = int(self.g.device_arrays()[1][j].item())
            details[3] = f"edge ({u}, {w}) spans levels {int(levels[u])} and {int(levels[w])}"
        if bad[4] >= 0:
            v = int(bad[4])
            if par(v) >= 0:
                details[4] = f"vertex {v} is reached but outside the source component"
            else:
                details[4] = f"vertex {v} is in the source component but unreached"
        checks = [CheckResult(name, bool(bad[i] < 0), details[i]) for i, name in enumerate(CHECK_NAMES)]
        return ValidationReport(passed=all(c.passed for c in checks), checks=checks, derived_levels=levels)


def validate(g: CsrGraph, source: int, parent, edge_list: EdgeList | None = None) -> ValidationReport:
    """One-shot validation (validate.py:228-235)."""
    return Validator(g, edge_list=edge_list).validate(source, parent)

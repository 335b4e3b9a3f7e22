"""Host side of K6 (csrc/k_nextuse.cu): predicted next use of cached blocks from the agent
workflow DAG (path_analysis.cpp:257-290, 408-444, 547-557).

The workflow-graph ingestion itself (parsing path expressions, locating a request's cursor
from its invocation history) stays on the host as BASELINE.json prescribes; what crosses
the C-ABI is the flattened expression (pyg_path_node, preorder) and each live workflow's
cursor frames (PathCursor::frames()).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import check

PATH_NODE_DTYPE = np.dtype([("kind", "<i4"), ("role", "<i4"), ("min", "<i4"), ("max", "<i4"),
                            ("p_continue", "<f8"), ("p", "<f8"), ("child", "<i4"),
                            ("ch_begin", "<i4"), ("ch_end", "<i4"), ("pad", "<i4")])
assert PATH_NODE_DTYPE.itemsize == 48


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


class PathTable:
    """Flattened path expressions resident on the device (one or several concatenated;
    node ids are global to the table)."""

    def __init__(self, table: dict, device="cuda"):
        n = len(table["kind"])
        a = np.zeros(n, PATH_NODE_DTYPE)
        for k in ("kind", "role", "min", "max", "p_continue", "p", "child", "ch_begin", "ch_end"):
            a[k] = table[k]
        self.n_nodes = n
        self.nodes = torch.from_numpy(a.view(np.uint8).copy()).to(device)
        ch = np.asarray(table["ch_list"] or [0], np.int32)
        self.ch_list = torch.from_numpy(ch).to(device)


def cursors_csr(frames_list, device="cuda"):
    off = np.zeros(len(frames_list) + 1, np.int32)
    np.cumsum([len(f) for f in frames_list], out=off[1:])
    flat = np.asarray([x for f in frames_list for x in f] or [(0, 0)], np.int32).reshape(-1, 2)
    return (torch.from_numpy(off).to(device), torch.from_numpy(flat[:, 0].copy()).to(device),
            torch.from_numpy(flat[:, 1].copy()).to(device))


def next_use(ctx, table: PathTable, frames_list, n_roles: int, device="cuda"):
    """-> (dist [n_cursors, n_roles] float64 with NaN for nullopt, future masks uint64)."""
    nc = len(frames_list)
    off, node, prog = cursors_csr(frames_list, device)
    dist = torch.empty((max(nc, 1), n_roles), dtype=torch.float64, device=device)
    fut = torch.zeros(max(nc, 1), dtype=torch.int64, device=device)
    check(_lib._lib.pyg_next_use_dev(ctx.h, _p(table.nodes), table.n_nodes, _p(table.ch_list), nc,
                                     _p(off), _p(node), _p(prog), n_roles, _p(dist), _p(fut)))
    return dist[:nc], fut[:nc]


def block_next_use(ctx, replica, tier, wf_cursor: torch.Tensor, dist: torch.Tensor):
    """Predicted next use of every block of (replica, tier), in id order."""
    n_roles = dist.shape[1]
    cap = 1 << 20
    out = torch.empty(cap, dtype=torch.float64, device=dist.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=dist.device)
    check(_lib._lib.pyg_block_next_use_dev(ctx.h, replica, tier, _p(wf_cursor),
                                           int(wf_cursor.numel()), _p(dist), n_roles, _p(out),
                                           cap, _p(cnt)))
    return out[:int(cnt.item())]


def registry_from_cursors(ctx, wf: torch.Tensor, cursor: torch.Tensor, future: torch.Tensor,
                          current_role: torch.Tensor | None = None, max_wf=None):
    max_wf = int(wf.max().item()) if max_wf is None and wf.numel() else (max_wf or 0)
    check(_lib._lib.pyg_registry_from_cursors_dev(ctx.h, int(wf.numel()), max_wf, _p(wf),
                                                  _p(cursor), _p(future), _p(current_role)))

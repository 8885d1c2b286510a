"""Communication metering of the reference (comm.hpp), host side.

The reference meters its simulated node messages in a CommLedger (comm.hpp:45-107)
written by the solvers every iteration (solvers.hpp:111,128,219-224,358-369,400).
On the B200 the exchanges are device reductions / NCCL collectives; the ledger is
filled with exactly the element counts the reference records so SolveReport.ledger
stays comparable.  The closed form is comm.hpp:128-155.
"""
from __future__ import annotations

import enum

import numpy as np

from .errors import ParameterError, PartitionError


class Method(enum.Enum):
    Consensus = "consensus"
    Sectioning = "sectioning"
    Hybrid = "hybrid"


class Convention(enum.Enum):
    SenderOnceBroadcast = "sender_once_broadcast"
    PerLink = "per_link"


class Counts:
    __slots__ = ("received", "sent")

    def __init__(self, received: int = 0, sent: int = 0):
        self.received = int(received)
        self.sent = int(sent)

    def total(self) -> int:
        return self.received + self.sent


class CommLedger:
    """Per-node, per-iteration element counts (comm.hpp:45-107)."""

    def __init__(self):
        self._cells = np.zeros((0, 0, 3), dtype=np.uint64)  # recv, sent_once, sent_links

    def _grow(self, node: int, iteration: int) -> None:
        n, k, _ = self._cells.shape
        if node >= n or iteration >= k:
            new = np.zeros((max(n, node + 1), max(k, iteration + 1), 3), dtype=np.uint64)
            new[:n, :k] = self._cells
            self._cells = new

    def record_recv(self, node: int, iteration: int, elements: int) -> None:
        self._grow(node, iteration)
        self._cells[node, iteration, 0] += np.uint64(elements)

    def record_send(self, node: int, iteration: int, elements: int) -> None:
        self._grow(node, iteration)
        self._cells[node, iteration, 1] += np.uint64(elements)
        self._cells[node, iteration, 2] += np.uint64(elements)

    def record_broadcast(self, node: int, iteration: int, elements: int, peers: int) -> None:
        self._grow(node, iteration)
        self._cells[node, iteration, 1] += np.uint64(elements)
        self._cells[node, iteration, 2] += np.uint64(elements * peers)

    def node_count(self) -> int:
        return int(self._cells.shape[0])

    def iteration_count(self) -> int:
        return int(self._cells.shape[1])

    def empty(self) -> bool:
        return self._cells.shape[0] == 0

    def counts(self, node: int, iteration: int,
               convention: Convention = Convention.SenderOnceBroadcast) -> Counts:
        if node >= self._cells.shape[0] or iteration >= self._cells.shape[1]:
            return Counts()
        c = self._cells[node, iteration]
        return Counts(c[0], c[1] if convention == Convention.SenderOnceBroadcast else c[2])

    def as_array(self) -> np.ndarray:
        """(nodes, iterations, 3): received, sent (sender-once), sent (per-link)."""
        return self._cells.copy()

    # -- bulk filling with the exact per-iteration records of each solver ----------
    @classmethod
    def for_solve(cls, method: str, row_bounds, col_bounds, iterations: int) -> "CommLedger":
        led = cls()
        if method == "reference" or iterations == 0:
            return led
        M, N = len(row_bounds) - 1, len(col_bounds) - 1
        rows = np.diff(np.asarray(row_bounds, dtype=np.uint64))
        cols = np.diff(np.asarray(col_bounds, dtype=np.uint64))
        n_meas, n_pix = int(row_bounds[-1]), int(col_bounds[-1])
        if method == "consensus":  # solvers.hpp:109-112 recv v, :128 send u+s
            cell = np.array([n_pix, n_pix, n_pix], dtype=np.uint64)
            led._cells = np.broadcast_to(cell, (M, iterations, 3)).copy()
        elif method == "sectioning":  # solvers.hpp:218-225
            cell = np.array([(N - 1) * n_meas, n_meas, n_meas * (N - 1)], dtype=np.uint64)
            led._cells = np.broadcast_to(cell, (N, iterations, 3)).copy()
        elif method == "hybrid":  # solvers.hpp:354-372, 398-402
            c = np.zeros((M * N, 3), dtype=np.uint64)
            for i in range(M):
                for j in range(N):
                    rl, cl = rows[i], cols[j]
                    c[i * N + j] = [cl + (N - 1) * rl, rl + cl, rl * (N - 1) + cl]
            led._cells = np.broadcast_to(c[:, None, :], (M * N, iterations, 3)).copy()
        else:
            raise ParameterError(f"unknown method {method}")
        return led


def _require_divides(d: int, total: int, what: str) -> None:
    if d == 0 or total % d != 0:
        raise PartitionError(f"per_node_elements: {d} does not divide {total} {what}")


def per_node_elements(method: Method, n_pix: int, n_meas: int, m: int, n: int) -> int:
    """Closed form of comm.hpp:128-148 (SenderOnceBroadcast)."""
    if n_pix == 0 or n_meas == 0 or m == 0 or n == 0:
        raise ParameterError("per_node_elements: sizes and divisions must be positive")
    if method == Method.Consensus:
        _require_divides(m, n_meas, "rows")
        return 2 * n_pix
    if method == Method.Sectioning:
        _require_divides(n, n_pix, "columns")
        return n * n_meas
    _require_divides(m, n_meas, "rows")
    _require_divides(n, n_pix, "columns")
    return n * (n_meas // m) + 2 * (n_pix // n)


def reduction_vs_consensus(method: Method, n_pix: int, n_meas: int, m: int, n: int) -> float:
    """comm.hpp:151-155."""
    return 100.0 * (1.0 - per_node_elements(method, n_pix, n_meas, m, n) / (2.0 * n_pix))

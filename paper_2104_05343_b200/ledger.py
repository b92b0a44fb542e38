"""Communication / compute ledger of the mesh (summagrid mesh.py:91-208, 385-419, 521-550).

Accounting only — it never affects results. Every collective the mesh runs is
charged with the reference's cost model, in units of beta x scalars:

* broadcast / reduce: binomial tree over the group, log2(g) * beta * n per
  member; every tree edge sends n scalars (intra- or inter-node by placement);
* all-reduce: ring, 2 * beta * (g - 1) * n / g per member; every member
  forwards 2 (g - 1) n / g scalars to its ring successor in 2 (g - 1) messages;

plus local multiply-accumulates per position. On the dist backend every
process keeps the same global ledger (the charges are deterministic functions
of the call sequence). The measured B200 counterpart is the panel-byte
accounting of the roofline (bench.py / DESIGN.md).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

COUNTERS = ("broadcast_cost", "reduce_cost", "allreduce_cost", "scalars_sent_internode", "scalars_sent_intranode",
            "macs", "messages_sent")


class CommLedger:
    """Per-position monotone counters plus per-(tag, kind) cost splits."""

    def __init__(self, p: int) -> None:
        self.p = p
        self.broadcast_cost = np.zeros(p)
        self.reduce_cost = np.zeros(p)
        self.allreduce_cost = np.zeros(p)
        self.scalars_sent_internode = np.zeros(p, dtype=np.int64)
        self.scalars_sent_intranode = np.zeros(p, dtype=np.int64)
        self.macs = np.zeros(p, dtype=np.int64)
        self.messages_sent = np.zeros(p, dtype=np.int64)
        self.cost_by_tag: dict[tuple[str, str], np.ndarray] = {}

    def _tag_array(self, tag: str, kind: str) -> np.ndarray:
        return self.cost_by_tag.setdefault((tag, kind), np.zeros(self.p))

    def snapshot(self) -> "CommReport":
        return CommReport(self.p, *(getattr(self, c).copy() for c in COUNTERS),
                          cost_by_tag={k: v.copy() for k, v in self.cost_by_tag.items()})

    # ---------------------------------------------------------------- charging
    def _edge(self, node_of, sender: int, receiver: int, n: int) -> None:
        if node_of(sender) == node_of(receiver):
            self.scalars_sent_intranode[sender] += n
        else:
            self.scalars_sent_internode[sender] += n
        self.messages_sent[sender] += 1

    def charge_tree(self, group: Sequence[int], root_pos: int, n: int, beta: float, tag: str, kind: str,
                    node_of) -> None:
        """Broadcast (data root -> leaves) or reduce (leaves -> root) over a binomial tree."""
        g = len(group)
        cost = math.log2(g) * beta * n if g > 1 else 0.0
        total = self.broadcast_cost if kind == "broadcast" else self.reduce_cost
        tagged = self._tag_array(tag, kind)
        for dev in group:
            total[dev] += cost
            tagged[dev] += cost
        step = 1
        while step < g:  # binomial tree in group order rotated to the root
            for vr in range(step):
                if vr + step < g:
                    parent, child = group[(vr + root_pos) % g], group[(vr + step + root_pos) % g]
                    if kind == "broadcast":
                        self._edge(node_of, parent, child, n)
                    else:
                        self._edge(node_of, child, parent, n)
            step *= 2

    def charge_ring(self, group: Sequence[int], n: int, beta: float, tag: str, node_of) -> None:
        g = len(group)
        cost = 2.0 * beta * (g - 1) * n / g if g > 1 else 0.0
        tagged = self._tag_array(tag, "allreduce")
        for dev in group:
            self.allreduce_cost[dev] += cost
            tagged[dev] += cost
        if g > 1:
            sent = 2 * (g - 1) * n // g if n % g == 0 else int(round(2 * (g - 1) * n / g))
            for pos, dev in enumerate(group):
                nxt = group[(pos + 1) % g]
                if node_of(dev) == node_of(nxt):
                    self.scalars_sent_intranode[dev] += sent
                else:
                    self.scalars_sent_internode[dev] += sent
                self.messages_sent[dev] += 2 * (g - 1)


@dataclass
class CommReport:
    """Immutable snapshot of a ledger with delta / comparison helpers (mesh.py:144-200)."""

    p: int
    broadcast_cost: np.ndarray
    reduce_cost: np.ndarray
    allreduce_cost: np.ndarray
    scalars_sent_internode: np.ndarray
    scalars_sent_intranode: np.ndarray
    macs: np.ndarray
    messages_sent: np.ndarray
    cost_by_tag: dict = field(default_factory=dict)

    def minus(self, earlier: "CommReport") -> "CommReport":
        zeros = np.zeros(self.p)
        tags = set(self.cost_by_tag) | set(earlier.cost_by_tag)
        return CommReport(self.p, *(getattr(self, c) - getattr(earlier, c) for c in COUNTERS),
                          cost_by_tag={k: self.cost_by_tag.get(k, zeros) - earlier.cost_by_tag.get(k, zeros)
                                       for k in tags})

    def tag_cost(self, tag: str, kinds: Iterable[str] = ("broadcast", "reduce", "allreduce")) -> np.ndarray:
        total = np.zeros(self.p)
        for kind in kinds:
            arr = self.cost_by_tag.get((tag, kind))
            if arr is not None:
                total = total + arr
        return total

    def comm_cost(self) -> np.ndarray:
        return self.broadcast_cost + self.reduce_cost + self.allreduce_cost

    def equals(self, other: "CommReport") -> bool:
        if not all(np.array_equal(getattr(self, c), getattr(other, c)) for c in COUNTERS):
            return False
        if set(self.cost_by_tag) != set(other.cost_by_tag):
            return False
        return all(np.array_equal(v, other.cost_by_tag[k]) for k, v in self.cost_by_tag.items())


def placement_traffic(report: CommReport) -> dict[str, int]:
    """Scalars crossing node boundaries vs staying inside a node (mesh.py:203-208)."""
    return {"internode": int(report.scalars_sent_internode.sum()),
            "intranode": int(report.scalars_sent_intranode.sum())}


def ledger_report(mesh) -> CommReport:
    """Side-effect-free snapshot of the mesh's counters (mesh.py:521-523)."""
    return mesh.ledger.snapshot()


def ledger_csv(report: CommReport, cols: int | None = None) -> str:
    """rank_row,rank_col,counter_name,value rows, positions in flat order (mesh.py:534-550);
    cost counters in repr float form, the rest integers."""
    c = cols or int(math.isqrt(report.p))
    lines = ["rank_row,rank_col,counter_name,value"]
    floats = {"broadcast_cost", "reduce_cost", "allreduce_cost"}
    for flat in range(report.p):
        for name in COUNTERS:
            val = getattr(report, name)[flat]
            lines.append(f"{flat // c},{flat % c},{name},{repr(float(val)) if name in floats else str(int(val))}")
    return "\n".join(lines) + "\n"

"""Pure-Python restatement of the reference's discrete-event device engine
(device.cpp:74-311) for small cases.

TEST INFRASTRUCTURE ONLY (see oracle/policy.py). Reproduces: exact-rational
per-TPC slot capacity (:94-119), priority-ordered residency (:137-155),
greedy refill with no bypass (:188-206), prelude per block when atomized
(:184), pause (:165-171), (t, seq) event order with one shared seq counter
(:232-262). Used to cross-check the C++ replay engine on randomized small
submissions (tests/test_oracle.py).
"""
from __future__ import annotations

import heapq
from fractions import Fraction

from .policy import block_latency


class Engine:
    def __init__(self, tpcs: int, fmax: int = 1410):
        self.fmax = fmax
        self.now = 0
        self.seq = 0
        self.events: list = []
        self.kernels: list[dict] = []
        self.atoms: list[dict] = []
        self.resident = [[] for _ in range(tpcs)]
        self.load = [Fraction(0) for _ in range(tpcs)]
        self.completions: list[tuple[int, int, int]] = []  # (atom, tag, time)
        self.executed: list[int] = []

    def register_kernel(self, blocks: int, d0: int, s: float, occ: int) -> int:
        self.kernels.append(dict(blocks=blocks, d0=d0, s=s, occ=occ, prelude=500))
        self.executed.append(0)
        return len(self.kernels) - 1

    def _push(self, t, kind, tpc=0, atom=0):
        heapq.heappush(self.events, (t, self.seq, kind, tpc, atom))
        self.seq += 1

    def submit(self, kid: int, lo: int, hi: int, tpcs: list[int], prio: int,
               atomized: bool, tag: int) -> int:
        a = dict(kid=kid, next=lo, end=hi, run=0, tpcs=sorted(tpcs), prio=prio,
                 seq=self.seq, atomized=atomized, paused=False, done=False, tag=tag)
        self.seq += 1
        self.atoms.append(a)
        aid = len(self.atoms) - 1
        for t in a["tpcs"]:
            res = self.resident[t]
            pos = len(res)
            for i, o in enumerate(res):
                oa = self.atoms[o]
                if oa["prio"] < prio or (oa["prio"] == prio and oa["seq"] > a["seq"]):
                    pos = i
                    break
            res.insert(pos, aid)
        for t in a["tpcs"]:
            self._fill(t)
        return aid

    def pause(self, aid: int, paused: bool) -> None:
        a = self.atoms[aid]
        if a["done"] or a["paused"] == paused:
            return
        a["paused"] = paused
        if not paused:
            for t in a["tpcs"]:
                self._fill(t)

    def _fill(self, t: int) -> None:
        while True:
            pick = next((i for i in self.resident[t]
                         if not self.atoms[i]["paused"] and self.atoms[i]["next"] < self.atoms[i]["end"]),
                        None)
            if pick is None:
                return
            a = self.atoms[pick]
            k = self.kernels[a["kid"]]
            if self.load[t] + Fraction(1, k["occ"]) > 1:
                return
            self.load[t] += Fraction(1, k["occ"])
            a["run"] += 1
            a["next"] += 1
            self.executed[a["kid"]] += 1
            d = block_latency(k["d0"], k["s"], self.fmax, self.fmax)
            if a["atomized"]:
                d += k["prelude"]
            self._push(self.now + d, 0, t, pick)

    def call(self, t: int, fn) -> None:
        heapq.heappush(self.events, (t, self.seq, 2, 0, fn))
        self.seq += 1

    def run(self) -> None:
        while self.events:
            t, _, kind, tpc, x = heapq.heappop(self.events)
            self.now = t
            if kind == 2:
                x()
                continue
            a = self.atoms[x]
            self.load[tpc] -= Fraction(1, self.kernels[a["kid"]]["occ"])
            a["run"] -= 1
            self._fill(tpc)
            if a["run"] == 0 and a["next"] == a["end"] and not a["done"]:
                a["done"] = True
                for tt in a["tpcs"]:
                    self.resident[tt] = [i for i in self.resident[tt] if i != x]
                self.completions.append((x, a["tag"], t))

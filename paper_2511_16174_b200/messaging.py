"""Trace events and the communication ledger (mirrors pipeevd/messaging.py:22-167).

On the B200 path these are populated from CUDA-event stage times and from the words the NCCL
collectives (or, on one GPU, the equivalent device-side hand-offs) move.
"""
from __future__ import annotations

import json
import threading
from dataclasses import asdict, dataclass

HOST = -1
BROADCAST = -2
TRACE_STAGES = ("SBR", "BC", "SBR-Back", "BC-Back", "Solver", "FinalMultiply", "Comm")


@dataclass
class TraceEvent:
    worker: int
    stage: str
    block: int
    t_start: int
    t_end: int
    words: int = 0

    def __post_init__(self):
        if self.stage not in TRACE_STAGES:
            raise ValueError(f"unknown trace stage {self.stage!r}")
        if self.t_end < self.t_start:
            raise ValueError("event ends before it starts")

    @property
    def duration(self) -> int:
        return self.t_end - self.t_start


class TraceLog:
    """Thread-safe append-only event collection (messaging.py:71-108)."""

    def __init__(self):
        self._events: list[TraceEvent] = []
        self._lock = threading.Lock()

    def add(self, worker, stage, block, t_start, t_end, words=0) -> TraceEvent:
        ev = TraceEvent(int(worker), stage, int(block), int(t_start), int(t_end), int(words))
        with self._lock:
            self._events.append(ev)
        return ev

    def events(self) -> list[TraceEvent]:
        with self._lock:
            evs = list(self._events)
        return sorted(evs, key=lambda e: (e.t_start, e.t_end, e.worker, e.stage))

    def __len__(self) -> int:
        with self._lock:
            return len(self._events)

    def to_ndjson(self, path) -> None:
        with open(path, "w") as fh:
            for ev in self.events():
                fh.write(json.dumps(asdict(ev)) + "\n")

    @staticmethod
    def from_ndjson(path) -> list[TraceEvent]:
        out = []
        with open(path) as fh:
            for line in fh:
                line = line.strip()
                if line:
                    out.append(TraceEvent(**json.loads(line)))
        return sorted(out, key=lambda e: (e.t_start, e.t_end, e.worker, e.stage))


class CommLedger:
    """FP64 words and messages per (src, dst, stage) (messaging.py:111-167)."""

    def __init__(self):
        self._words: dict = {}
        self._msgs: dict = {}
        self._lock = threading.Lock()

    def record(self, src: int, dst: int, stage: str, words: int) -> None:
        words = int(words)
        if words < 0:
            raise ValueError("message word counts only increase")
        key = (int(src), int(dst), stage)
        with self._lock:
            self._words[key] = self._words.get(key, 0) + words
            self._msgs[key] = self._msgs.get(key, 0) + 1

    def _select(self, table, stage, src, dst) -> int:
        with self._lock:
            items = list(table.items())
        return sum(v for (s, d, st), v in items
                   if (stage is None or st == stage) and (src is None or s == src)
                   and (dst is None or d == dst))

    def words(self, stage=None, src=None, dst=None) -> int:
        return self._select(self._words, stage, src, dst)

    def messages(self, stage=None, src=None, dst=None) -> int:
        return self._select(self._msgs, stage, src, dst)

    @property
    def total_words(self) -> int:
        return self.words()

    def stages(self) -> list[str]:
        with self._lock:
            return sorted({k[2] for k in self._words})

    def to_csv(self) -> str:
        with self._lock:
            items = sorted(self._words.items())
        return "src,dst,stage,words\n" + "".join(f"{s},{d},{st},{v}\n" for (s, d, st), v in items)

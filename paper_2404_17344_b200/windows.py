"""Feature-window arrangement (the sub-kernel index sets).

Mirrors ``addkern.windows.WindowSet`` (/root/reference/pkg/src/addkern/windows.py:14-76):
windows are strictly ascending tuples of 1-based feature indices, each of
length 1..d_max with d_max <= 3, indices may repeat across windows, and the
JSON form is ``{"windows": [...], "d_max": k, "metadata": {...}}``.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Iterator


def _validate(windows: tuple, d_max: int) -> None:
    if not (1 <= d_max <= 3):
        raise ValueError(f"d_max must be in 1..3, got {d_max}")
    if not windows:
        raise ValueError("a WindowSet needs at least one window")
    for win in windows:
        if len(win) < 1 or len(win) > d_max:
            raise ValueError(f"window {win} longer than d_max={d_max}")
        if min(win) < 1:
            raise ValueError(f"window {win} has non-positive index")
        if any(b <= a for a, b in zip(win, win[1:])):
            raise ValueError(f"window {win} must be strictly ascending")


@dataclass(frozen=True)
class WindowSet:
    """Ordered collection of feature windows (1-based, ascending)."""

    windows: tuple
    d_max: int
    metadata: dict = field(default_factory=dict, compare=False)

    def __post_init__(self):
        normalised = tuple(tuple(int(i) for i in win) for win in self.windows)
        object.__setattr__(self, "windows", normalised)
        _validate(normalised, self.d_max)

    def __len__(self) -> int:
        return len(self.windows)

    def __iter__(self) -> Iterator[tuple]:
        return iter(self.windows)

    @property
    def n_windows(self) -> int:
        return len(self.windows)

    @property
    def lengths(self) -> tuple:
        return tuple(map(len, self.windows))

    def columns(self, window) -> list:
        """0-based numpy columns of one window (reference windows.py:57-59)."""
        return [int(i) - 1 for i in window]

    def max_feature(self) -> int:
        return max(i for win in self.windows for i in win)

    def to_json(self) -> str:
        body = {"d_max": self.d_max, "metadata": self.metadata,
                "windows": [list(win) for win in self.windows]}
        return json.dumps(body, indent=2, sort_keys=True)

    @classmethod
    def from_json(cls, text: str) -> "WindowSet":
        body = json.loads(text)
        return cls(tuple(tuple(win) for win in body["windows"]), int(body["d_max"]),
                   body.get("metadata", {}))


def singleton_windows(d: int) -> WindowSet:
    """{1}, {2}, ..., {d} (reference windows.py:79-81)."""
    return WindowSet(tuple((i + 1,) for i in range(d)), d_max=1)


def consec_windows(d: int, d_max: int) -> WindowSet:
    """Consecutive, non-overlapping windows of length d_max covering 1..d.

    The arrangement the BASELINE configurations use (reference
    grouping.py:93-99); a shorter last window takes the remainder.
    """
    if d < 1:
        raise ValueError("d must be positive")
    wins = []
    start = 1
    while start <= d:
        stop = min(start + d_max - 1, d)
        wins.append(tuple(range(start, stop + 1)))
        start = stop + 1
    return WindowSet(tuple(wins), d_max=d_max, metadata={"technique": "consec"})

"""Backend selector kept for API compatibility (kernel_exec.py:39-66).

The reference's `place=` parameter chooses between its sequential and threaded
CPU team emulations.  Here every operator runs on the CUDA device through
libb200hydro.so; `ExecPlace` is accepted and validated so scripts written
against the reference keep working, and `ExecPlace.parse` additionally accepts
"cuda" / "cuda:N".  There is no multi-backend dispatch.
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["ExecPlace"]


@dataclass(frozen=True)
class ExecPlace:
    workers: int = 0  # reference semantics: 0 = sequential, N = threads (informational here)
    device: int = 0

    @staticmethod
    def sequential() -> "ExecPlace":
        return ExecPlace(0)

    @staticmethod
    def threaded(workers: int) -> "ExecPlace":
        if workers < 1:
            raise ValueError("worker count must be >= 1")
        return ExecPlace(workers)

    @staticmethod
    def cuda(device: int = 0) -> "ExecPlace":
        return ExecPlace(0, device)

    @property
    def is_threaded(self) -> bool:
        return self.workers > 0

    @staticmethod
    def parse(text: str) -> "ExecPlace":
        """'seq', 'threads:N' (reference spellings) or 'cuda' / 'cuda:N'."""
        if text == "seq":
            return ExecPlace.sequential()
        if text.startswith("threads:"):
            return ExecPlace.threaded(int(text.split(":", 1)[1]))
        if text == "cuda":
            return ExecPlace.cuda(0)
        if text.startswith("cuda:"):
            return ExecPlace.cuda(int(text.split(":", 1)[1]))
        raise ValueError(f"unknown exec place {text!r} (want 'seq', 'threads:N' or 'cuda[:N]')")


SEQ = ExecPlace.sequential()

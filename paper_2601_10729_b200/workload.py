"""Synthetic request traces and the canonical trace file format.

Mirrors /root/reference/pkg/src/kvsim/workload.py (gamma inter-arrivals with
shape 1/cv^2, log-normal or fixed lengths; CSV records after ``#key=value``
metadata).  The generator consumes the numpy ``default_rng`` stream in the
reference's order, so the same seed yields the same trace - the config-3
mixed-length trace of BASELINE.json is produced here.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from pathlib import Path

import numpy as np


@dataclass(frozen=True)
class TraceRequest:
    arrival_ms: int
    prompt_tokens: int
    output_tokens: int

    def __post_init__(self) -> None:
        if self.arrival_ms < 0:
            raise ValueError("arrival_ms must be >= 0")
        if min(self.prompt_tokens, self.output_tokens) < 1:
            raise ValueError("token counts must be >= 1")


@dataclass(frozen=True)
class Trace:
    requests: tuple[TraceRequest, ...]
    metadata: dict = field(default_factory=dict)

    def __post_init__(self) -> None:
        arrivals = [r.arrival_ms for r in self.requests]
        if any(b < a for a, b in zip(arrivals, arrivals[1:])) or (arrivals and arrivals[0] < 0):
            raise ValueError("arrival times must be non-decreasing")

    def __eq__(self, other) -> bool:
        if not isinstance(other, Trace):
            return NotImplemented
        return (self.requests, self.metadata) == (other.requests, other.metadata)


@dataclass(frozen=True)
class LengthSpec:
    """Prompt/output length distribution: ``lognormal`` or ``fixed``."""

    kind: str = "lognormal"
    prompt_median: float = 512.0
    prompt_sigma: float = 0.9
    output_median: float = 80.0
    output_sigma: float = 0.7
    max_prompt: int = 4096
    max_output: int = 512
    fixed_prompt: int = 512
    fixed_output: int = 64

    def __post_init__(self) -> None:
        if self.kind not in ("lognormal", "fixed"):
            raise ValueError(f"unknown length spec kind {self.kind!r}")
        if self.kind == "lognormal":
            if min(self.prompt_median, self.output_median) < 1:
                raise ValueError("medians must be >= 1")
            if min(self.prompt_sigma, self.output_sigma) < 0:
                raise ValueError("sigmas must be >= 0")
        if min(self.max_prompt, self.max_output) < 1:
            raise ValueError("length caps must be >= 1")


def _lengths(rng, spec: LengthSpec, count: int):
    if spec.kind == "fixed":
        return (np.full(count, spec.fixed_prompt, dtype=np.int64),
                np.full(count, spec.fixed_output, dtype=np.int64))
    raw_p = rng.lognormal(np.log(spec.prompt_median), spec.prompt_sigma, count)
    raw_o = rng.lognormal(np.log(spec.output_median), spec.output_sigma, count)
    clip = lambda x, hi: np.clip(np.rint(x), 1, hi).astype(np.int64)  # noqa: E731
    return clip(raw_p, spec.max_prompt), clip(raw_o, spec.max_output)


def _metadata(seed, rate, cv, spec: LengthSpec) -> dict:
    meta = {"seed": str(seed), "rate": repr(rate), "cv": repr(cv), "kind": spec.kind}
    if spec.kind == "lognormal":
        meta.update(prompt_median=repr(spec.prompt_median), prompt_sigma=repr(spec.prompt_sigma),
                    output_median=repr(spec.output_median), output_sigma=repr(spec.output_sigma),
                    max_prompt=str(spec.max_prompt), max_output=str(spec.max_output))
    else:
        meta.update(fixed_prompt=str(spec.fixed_prompt), fixed_output=str(spec.fixed_output))
    return meta


def generate(seed: int, rate: float, cv: float, length_spec: LengthSpec, count: int) -> Trace:
    """Deterministic trace: gamma gaps with mean 60000/rate ms and shape 1/cv^2."""
    if rate <= 0:
        raise ValueError("rate must be > 0 requests/min")
    if cv <= 0:
        raise ValueError("cv must be > 0")
    if count < 0:
        raise ValueError("count must be >= 0")
    rng = np.random.default_rng(seed)
    shape = 1.0 / (cv * cv)
    gaps = rng.gamma(shape, (60000.0 / rate) / shape, size=count)
    arrivals = np.cumsum(gaps)
    prompts, outputs = _lengths(rng, length_spec, count)
    reqs = tuple(TraceRequest(int(round(a)), int(p), int(o))
                 for a, p, o in zip(arrivals, prompts, outputs))
    return Trace(reqs, _metadata(seed, rate, cv, length_spec))


class TraceFormatError(ValueError):
    pass


def serialize(trace: Trace) -> str:
    header = " ".join(f"{key}={trace.metadata[key]}" for key in sorted(trace.metadata))
    out = [f"# {header}".rstrip(), "# fields=arrival_ms,prompt_tokens,output_tokens"]
    out.extend(f"{r.arrival_ms},{r.prompt_tokens},{r.output_tokens}" for r in trace.requests)
    return "\n".join(out) + "\n"


def save(trace: Trace, path) -> None:
    Path(path).write_text(serialize(trace), encoding="utf-8")


def _parse_record(path, lineno: int, line: str, previous) -> TraceRequest:
    fields = line.split(",")
    if len(fields) != 3:
        raise TraceFormatError(f"{path}:{lineno}: expected 3 fields, got {len(fields)}")
    try:
        arrival, prompt, output = (int(f) for f in fields)
    except ValueError as exc:
        raise TraceFormatError(f"{path}:{lineno}: non-integer field ({exc})") from None
    if prompt < 1 or output < 1:
        raise TraceFormatError(f"{path}:{lineno}: token counts must be >= 1")
    if arrival < 0:
        raise TraceFormatError(f"{path}:{lineno}: arrival must be >= 0")
    if previous is not None and arrival < previous.arrival_ms:
        raise TraceFormatError(f"{path}:{lineno}: arrivals must be non-decreasing")
    return TraceRequest(arrival, prompt, output)


def load(path) -> Trace:
    reqs: list[TraceRequest] = []
    meta: dict = {}
    for lineno, raw in enumerate(Path(path).read_text(encoding="utf-8").splitlines(), start=1):
        line = raw.strip()
        if not line:
            continue
        if line.startswith("#"):
            for pair in line[1:].split():
                key, sep, value = pair.partition("=")
                if sep and key != "fields":
                    meta[key] = value
            continue
        reqs.append(_parse_record(path, lineno, line, reqs[-1] if reqs else None))
    return Trace(tuple(reqs), meta)

"""Chunk planning -- the reference's storage-cost model (Eqs. 2-7), re-parameterised for B200.

API-compatible with the reference's `planner.py` (`SystemParams` :47-76,
`ChunkPlan` :79-92, `compute_chunk_plan` :106-152, `with_overrides` :225-228).
On the CPU, MAGNUS sizes fine chunks so that the histogram, the offsets, two
write-combining lines per chunk and one dense accumulator stay in a core's
private L2.  On a B200 the private, software-managed level that plays that role
is a CTA's shared memory, so `detect_device_params` maps

    l2_bytes          := opt-in shared memory per block (227 KB on B200)
    cache_line_bytes  := 128 (L2 line; one coalesced store segment)
    memory_budget     := a fraction of free HBM (coarse-batch workspace cap)

The same `SystemParams` also selects the reference-visible behaviour of a call
(row categories, the per-chunk sort/dense accumulator choice and therefore the
summation association of every output value), so passing the reference's
host `SystemParams` reproduces the reference's result bit for bit.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, replace

from .errors import InputError

SYMBOLIC = "symbolic"
NUMERIC = "numeric"

# planner.py:41 -- above this coarse-chunk count the reference only warns
COARSE_CHUNKS_WARN = 1 << 13


def ceil_pow2(x: int) -> int:
    if x < 1:
        raise ValueError("ceil_pow2 requires x >= 1")
    return 1 << (int(x) - 1).bit_length()


def floor_pow2(x: int) -> int:
    if x < 1:
        raise ValueError("floor_pow2 requires x >= 1")
    return 1 << (int(x).bit_length() - 1)


def exact_log2(x: int) -> int:
    x = int(x)
    if x < 1 or x & (x - 1):
        raise ValueError(f"{x} is not a power of two")
    return x.bit_length() - 1


def round_pow2_of_sqrt(num: int, den: int) -> int:
    """Nearest power of two to sqrt(num/den) on the log2 scale, ties up (util.py:28-44)."""
    if num <= 0 or den <= 0:
        raise ValueError("num and den must be positive")
    if num < den:
        return 1
    k = (num // den).bit_length() // 2          # first guess, then correct exactly
    while k > 0 and num < den << (2 * k):
        k -= 1
    while num >= den << (2 * (k + 1)):
        k += 1
    if num >= den << (2 * k + 1):
        k += 1
    return 1 << k


@dataclass(frozen=True)
class SystemParams:
    cache_line_bytes: int = 64
    l2_bytes: int = 1 << 20
    memory_budget_bytes: int = 1 << 31
    histo_type_bytes: int = 4
    prefix_sum_type_bytes: int = 4
    val_bytes: int = 8

    def __post_init__(self):
        for name in ("cache_line_bytes", "l2_bytes", "memory_budget_bytes", "histo_type_bytes",
                     "prefix_sum_type_bytes", "val_bytes"):
            if getattr(self, name) <= 0:
                raise InputError(f"{name} must be positive")
        if self.cache_line_bytes & (self.cache_line_bytes - 1):
            raise InputError("cache_line_bytes must be a power of two")

    @property
    def s_chunk_fine(self) -> int:
        return self.histo_type_bytes + self.prefix_sum_type_bytes + 2 * self.cache_line_bytes

    def dense_accum_bytes(self, phase: str) -> int:
        return 1 if phase == SYMBOLIC else self.val_bytes + 1


@dataclass(frozen=True)
class ChunkPlan:
    phase: str
    plan_cols: int
    s_dense_accum: int
    s_chunk_fine: int
    n_chunks_fine: int
    chunk_len_fine: int
    shift_fine: int
    m_max_l2: int
    use_coarse: bool
    n_chunks_coarse: int
    chunk_len_coarse: int
    shift_coarse: int


def fine_level_storage(n_chunks: int, span: int, s_dense_accum: int, s_chunk_fine: int) -> int:
    """Eq. (2): accumulator slice plus per-chunk metadata."""
    return span * s_dense_accum // n_chunks + n_chunks * s_chunk_fine


def max_l2_cols(l2_bytes: int, s_dense_accum: int, s_chunk_fine: int) -> int:
    """Eq. (5): widest power-of-two span whose optimal fine level fits."""
    raw = l2_bytes * l2_bytes // (4 * s_dense_accum * s_chunk_fine)
    return floor_pow2(raw) if raw >= 1 else 1


def compute_chunk_plan(sys: SystemParams, m_c: int, phase: str, allow_coarse: bool = True) -> ChunkPlan:
    """Eqs. (3)-(7) for ``m_c`` output columns (reference planner.py:106-152).

    The coarse/fine decision always uses the symbolic accumulator cost (one
    byte per slot) so both phases agree on categories; only the fine chunk
    count uses the phase's own cost.
    """
    if m_c < 1:
        raise InputError("m_c must be >= 1")
    if phase not in (SYMBOLIC, NUMERIC):
        raise InputError(f"unknown phase {phase!r}")
    plan_cols = ceil_pow2(m_c)
    sda = sys.dense_accum_bytes(phase)
    scf = sys.s_chunk_fine
    m_max = max_l2_cols(sys.l2_bytes, sys.dense_accum_bytes(SYMBOLIC), scf)
    use_coarse = bool(allow_coarse and plan_cols > m_max)
    span = m_max if use_coarse else plan_cols
    n_fine = round_pow2_of_sqrt(span * sda, scf)
    min_len = max(1, sys.cache_line_bytes // 4)
    n_fine = max(1, min(n_fine, max(1, span // min_len), span))
    chunk_len = span // n_fine
    n_coarse, len_coarse = (plan_cols // m_max, m_max) if use_coarse else (1, plan_cols)
    if n_coarse > COARSE_CHUNKS_WARN:
        warnings.warn(f"{n_coarse} coarse chunks exceeds the measured reorder breaking point "
                      f"({COARSE_CHUNKS_WARN}); expect reduced throughput", stacklevel=2)
    return ChunkPlan(phase, plan_cols, sda, scf, n_fine, chunk_len, exact_log2(chunk_len), m_max, use_coarse,
                     n_coarse, len_coarse, exact_log2(len_coarse))


def detect_device_params(device=None, memory_budget_fraction: float = 0.25, val_bytes: int = 8) -> SystemParams:
    """B200 counterpart of the reference's host probe (`detect_system_params`, planner.py:179-222)."""
    import torch

    if not torch.cuda.is_available():
        raise InputError("no CUDA device: the B200 path has no CPU fallback")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    props = torch.cuda.get_device_properties(dev)
    smem = int(getattr(props, "shared_memory_per_block_optin", 0) or 232448)
    free, _total = torch.cuda.mem_get_info(dev)
    budget = max(1, int(free * memory_budget_fraction))
    return SystemParams(cache_line_bytes=128, l2_bytes=smem, memory_budget_bytes=budget, val_bytes=val_bytes)


def b200_default_params() -> SystemParams:
    """Device-independent stand-in for `detect_device_params` (no GPU needed): B200 numbers."""
    return SystemParams(cache_line_bytes=128, l2_bytes=232448, memory_budget_bytes=40 << 30)


def with_overrides(sys: SystemParams, **kwargs) -> SystemParams:
    updates = {k: v for k, v in kwargs.items() if v is not None}
    return replace(sys, **updates) if updates else sys

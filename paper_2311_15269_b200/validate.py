"""Schedule validation on the B200.

``validate_schedule_device(s)`` returns exactly the list the reference's
``validate_schedule`` (schedule.py:77-168) returns — same violations, kinds,
messages, instance tuples and order — with the per-device sort, overlap,
running-memory, dependency and negative-start checks in sm_100a kernels
(csrc/validate.cuh, C ABI ``tsl_validate``).  The host only checks the
instance set and formats the messages of flagged positions.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .placement import BlockInstance
from .schedule import Schedule, Violation

__all__ = ["validate_schedule_device"]


def _u8(n):
    return np.zeros(max(n, 1), dtype=np.uint8)


def validate_schedule_device(s: Schedule, initial_memory=None) -> list:
    p = s.placement
    K, D, N = p.num_stages, p.num_devices, s.num_microbatches
    found = []
    want = {BlockInstance(st, n) for st in range(K) for n in range(N)}
    have = set(s.entries)
    if want != have:  # structure (schedule.py:88-103)
        found.append(Violation(
            "structure",
            f"instance set mismatch (missing {sorted(want - have)[:4]}, extra {sorted(have - want)[:4]})"))
        return found
    starts = np.zeros(K * N, dtype=np.int64)
    for b, t in s.entries.items():
        starts[b.stage * N + b.mb] = t
    if starts.size and (starts.max() >= 2 ** 31 or starts.min() < -2 ** 31):
        raise ValueError("start times outside the device kernel's int32 range")
    starts = starts.astype(np.int32)
    dur = np.array([p.block(st).time_cost for st in range(K)], dtype=np.int32)
    mem = np.array([p.block(st).mem_delta for st in range(K)], dtype=np.int32)
    masks = np.array([sum(1 << d for d in p.block(st).devices) for st in range(K)], dtype=np.uint64)
    deps = sorted(p.deps)
    dep_arr = np.array([x for e in deps for x in e] or [0, 0], dtype=np.int32)
    dstages = [p.device_stages(d) for d in range(D)]
    max_e = max(len(ds) * N for ds in dstages) or 1
    P = 1
    while P < max_e:
        P <<= 1
    init = np.array(list(initial_memory) if initial_memory else [0] * D, dtype=np.int64)
    cap = p.mem_capacity
    count = np.zeros(1, dtype=np.int64)
    keys = np.zeros(D * P, dtype=np.uint64)
    ovf, memf = _u8(D * P), _u8(D * P)
    runs = np.zeros(D * P, dtype=np.int64)
    depf, negf = _u8(len(deps) * N), _u8(K * N)
    L = _native.lib()
    _native.check(L.tsl_validate(K, D, _native._ptr(dur), _native._ptr(mem), _native._ptr(masks),
                                 len(deps), _native._ptr(dep_arr), N, _native._ptr(starts),
                                 _native._ptr(init), int(cap), int(P), _native._ptr(count),
                                 _native._ptr(keys), _native._ptr(ovf), _native._ptr(memf),
                                 _native._ptr(runs), _native._ptr(depf), _native._ptr(negf)))
    if count[0] == 0 and not (initial_memory and any(v > cap for v in initial_memory)):
        return found
    for b, t in s.entries.items():  # negative starts, in entry order (schedule.py:104-106)
        if negf[b.stage * N + b.mb]:
            found.append(Violation("structure", f"{b} has negative start {t}", (b,)))

    def event(d, q):  # sorted position q of device d -> (start, stage, mb)
        k = int(keys[d * P + q])
        pos = k & 0xffffffff
        u = (k >> 32) ^ 0x80000000  # the start's two's-complement bits
        return u - (1 << 32) if u >= 1 << 31 else u, dstages[d][pos // N], pos % N

    for d in range(D):  # overlaps between sorted neighbours (schedule.py:110-125)
        e = len(dstages[d]) * N
        for q in np.nonzero(ovf[d * P:d * P + e])[0]:
            t0, a0, n0 = event(d, q)
            t1, a1, n1 = event(d, q + 1)
            found.append(Violation(
                "overlap", f"device {d}: ({a0},{n0})@{t0} overlaps ({a1},{n1})@{t1}",
                (BlockInstance(a0, n0), BlockInstance(a1, n1))))
    for d in range(D):  # running memory per equal-start group (schedule.py:128-153)
        e = len(dstages[d]) * N
        total = int(init[d])
        if total > cap:
            found.append(Violation("memory", f"device {d}: initial memory {total} > M"))
        for q in np.nonzero(memf[d * P:d * P + e])[0]:
            t, _, _ = event(d, q)
            g = q
            while g > 0 and event(d, g - 1)[0] == t:
                g -= 1
            insts = tuple(BlockInstance(a, n) for _, a, n in (event(d, x) for x in range(g, q + 1)))
            found.append(Violation(
                "memory", f"device {d}: running memory {int(runs[d * P + q])} > {cap} at t={t}",
                insts))
    for qi, (a, b) in enumerate(deps):  # dependencies (schedule.py:155-167)
        ta = p.block(a).time_cost
        for n in np.nonzero(depf[qi * N:(qi + 1) * N])[0]:
            sa = s.entries[BlockInstance(a, int(n))]
            sb = s.entries[BlockInstance(b, int(n))]
            found.append(Violation(
                "dependency", f"({a},{n}) ends at {sa + ta} after ({b},{n}) starts at {sb}",
                (BlockInstance(a, int(n)), BlockInstance(b, int(n)))))
    return found

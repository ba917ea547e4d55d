"""MapModel.audit on the device (lm_audit, csrc/lm_audit.cuh), formatted with the
reference's violation messages (pkg/src/localmap/mapmodel.py:304-353) and in its order:
points by id (dead-with-observations / dead keyframe / binding mismatch / counters), then
slots by keyframe insertion order and keypoint, then covisibility pairs by keyframe id."""

from __future__ import annotations

import ctypes as C

from . import _lib

_POINT, _SLOT, _COVIS = 0, 1, 2


def _message(r) -> tuple[tuple, str]:
    c = r.code
    if c == 1:
        return (_POINT, r.mp, 0, 0), f"dead map point {r.mp} retains observations"
    if c == 2:
        return (_POINT, r.mp, 1, r.kf_a), f"map point {r.mp} observes dead keyframe {r.kf_a}"
    if c == 3:
        return (_POINT, r.mp, 1, r.kf_a), f"binding mismatch: map point {r.mp} vs slot ({r.kf_a}, {r.kp})"
    if c == 4:
        return (_POINT, r.mp, 2, 0), f"scale_counts mismatch for map point {r.mp}"
    if c == 5:
        return (_POINT, r.mp, 3, 0), f"scale_counts sum mismatch for map point {r.mp}"
    if c == 6:
        return (_SLOT, r.kf_a, r.kp, 0), f"slot ({r.kf_a}, {r.kp}) bound to dead point {r.mp}"
    if c == 7:
        return (_SLOT, r.kf_a, r.kp, 0), f"slot ({r.kf_a}, {r.kp}) not in map point {r.mp} observations"
    a, b = sorted((r.kf_a, r.kf_b))
    return (_COVIS, a, b, 0), f"covisibility weight mismatch for pair ({a}, {b})"


def device_audit(model, cap: int = 1 << 14) -> list[str]:
    recs = (_lib.AuditRecord * cap)()
    n = C.c_int32()
    model.ctx.call("lm_audit", model.map, recs, cap, C.byref(n))
    got = [_message(recs[k]) for k in range(min(n.value, cap))]
    order = {k: i for i, k in enumerate(model._kfs)}  # slots: keyframe insertion order
    got.sort(key=lambda km: (km[0][0], order.get(km[0][1], km[0][1]) if km[0][0] == _SLOT else km[0][1])
             + km[0][2:])
    out = [m for _, m in got]
    if n.value > cap:
        out.append(f"... {n.value - cap} more violations")
    return out

"""Exhaustive-scan restatement of the reference split objective — oracle only.

Restates Eq. 10 as evaluated by kvoverlap.scheduler.layer_time
(scheduler.py:76-92) over every split l in [0, s'] (scan_split,
scheduler.py:176-188), with the byte/FLOP terms of costmodel.py:131-143,
169-176 and the affine timing of hwprofile.py:64-85, written out inline so
the product's closed-form solver is checked against an independent route.
Operation order matches the reference so values agree to the last bit.
"""

from __future__ import annotations

import math


def layer_total(h, b, p, q, seq, l, flops, eff, bw, lat, column):
    rec_flops = 4 * b * l * h * h
    v = flops * eff
    t_rec = 0.0 if rec_flops == 0 else (math.inf if v == 0 else rec_flops / v)
    kv_bytes = 2 * b * (seq - l) * h * q
    t_kv = 0.0 if kv_bytes == 0 else lat + kv_bytes / bw
    if column:
        act = b * l * h * p
        t_act = 0.0 if act == 0 else lat + act / bw
    else:
        t_act = 0.0
    return t_act + max(t_rec, t_kv), t_rec, t_kv, t_act


def scan(h, b, p, q, seq, flops, eff, bw, lat, mode):
    """(l, total, t_rec, t_kv, t_act) minimising the objective; smallest l on ties."""
    column = mode == "column"
    best = None
    for l in range(seq + 1):
        t = layer_total(h, b, p, q, seq, l, flops, eff, bw, lat, column)
        if best is None or t[0] < best[1]:
            best = (l,) + t
    return best

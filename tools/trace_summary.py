"""Summarise an RBFFD_TRACE file (per step and CTA: globaltimer at kernel
entry, dependency resolved (griddepcontrol.wait), ring fully issued, exit
after the CTA's epilogue).  Needs a library built with `make TRACE=1`.

    RBFFD_TRACE=/tmp/t.bin python bench.py --quick ...; python tools/trace_summary.py /tmp/t.bin
"""
import sys

import numpy as np


def runs(path):
    raw = np.fromfile(path, dtype=np.uint64)
    i = 0
    while i < raw.size:
        G, S = int(raw[i].astype(np.int64)), int(raw[i + 1])
        i += 2
        g = abs(G)
        yield G < 0, raw[i:i + g * S * 4].reshape(S, g, 4).astype(np.int64)
        i += g * S * 4


def summarise_loop(t):
    """Persistent loop (header grid < 0): per step and CTA: consumers start,
    CTA arrival at the grid barrier, release seen, chunks armed ahead."""
    S = t.shape[0]
    start, arr, rel, ahead = t[:, :, 0], t[:, :, 1], t[:, :, 2], t[:, :, 3]
    us = lambda x: f"{np.median(x) / 1e3:7.2f}"
    print(f"steps {S}  CTAs {t.shape[1]}  (persistent loop)")
    print(f"  period (last release to last release)     {us(np.diff(rel.max(1)))} us")
    print(f"  CTA work (start -> arrival), mean / max   {us((arr - start).mean(1))} / {us((arr - start).max(1))} us")
    print(f"  arrival spread (first -> last CTA)        {us(arr.max(1) - arr.min(1))} us")
    print(f"  barrier (last arrival -> first release)   {us(rel.min(1) - arr.max(1))} us")
    print(f"  release spread (first -> last CTA)        {us(rel.max(1) - rel.min(1))} us")
    print(f"  CTA idle at the barrier, mean             {us((rel - arr).mean(1))} us")
    if ahead.max() > 1000:  # part loop traces: longest halo wait of a warp (ns)
        print(f"  longest neighbour wait per CTA, mean / max {us(ahead.mean(1))} / {us(ahead.max(1))} us")
    else:
        print(f"  next-step chunks armed at arrival, mean   {np.median(ahead.mean(1)):7.2f}")


def summarise(t):
    S = t.shape[0]
    entry, wait, issued, exit_ = t[:, :, 0], t[:, :, 1], t[:, :, 2], t[:, :, 3]
    span = exit_.max(1) - wait.min(1)
    imb = exit_.max(1) - exit_.min(1)
    gap = wait.min(1)[1:] - exit_.max(1)[:-1]  # dependency resolution after the previous step's last CTA
    early = entry.min(1)[1:] - exit_.max(1)[:-1]  # next step's first CTA entry vs this step's end
    prod = issued.max(1) - wait.min(1)
    drain = (exit_ - issued).mean(1)  # per CTA: last chunk issued -> CTA done
    period = exit_.max(1)[1:] - exit_.max(1)[:-1]
    us = lambda x: f"{np.median(x) / 1e3:7.2f}"
    print(f"steps {S}  CTAs {t.shape[1]}")
    print(f"  period (last exit to last exit)          {us(period)} us")
    print(f"  compute span (first dep. resolved -> last exit) {us(span)} us")
    print(f"  exit imbalance (first -> last CTA exit)  {us(imb)} us")
    print(f"  dependency gap (last exit -> next first resolved) {us(gap)} us")
    print(f"  next step's first CTA entry vs last exit {us(early)} us (negative: PDL prelaunch)")
    print(f"  producer: ring issued (last CTA) after first resolved {us(prod)} us")
    print(f"  drain (CTA mean: last chunk issued -> exit) {us(drain)} us")


if __name__ == "__main__":
    for k, (loop, t) in enumerate(runs(sys.argv[1])):
        print(f"== run {k}")
        if t.shape[0] > 2:
            (summarise_loop if loop else summarise)(t[1:])  # the first step has no predecessor

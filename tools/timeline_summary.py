#!/usr/bin/env python3
"""Summarise a chrome-trace timeline written by `bench.py --config c5 --timeline PATH`
(not part of the product): per CUDA stream, the kernels, their busy time and the gaps;
how much of the routing kernels' time overlaps the beamforming kernels.

    python tools/timeline_summary.py gpurun_out/timeline_c5.json
"""
import collections
import json
import sys


def main():
    tr = json.load(open(sys.argv[1]))
    ev = [e for e in tr.get("traceEvents", []) if e.get("ph") == "X" and e.get("cat") == "kernel"]
    by_stream = collections.defaultdict(list)
    for e in ev:
        by_stream[e["args"].get("stream", e.get("tid"))].append((e["ts"], e["ts"] + e["dur"], e["name"]))
    span0 = min(t0 for v in by_stream.values() for t0, _, _ in v)
    span1 = max(t1 for v in by_stream.values() for _, t1, _ in v)
    print(f"step span {span1 - span0:.1f} us, {len(ev)} kernels")
    apply_iv = []
    for st, v in sorted(by_stream.items(), key=lambda x: str(x[0])):
        v.sort()
        busy = sum(t1 - t0 for t0, t1, _ in v)
        names = collections.Counter(n.split("<")[0].split("(")[0][-40:] for _, _, n in v)
        gaps = [v[i + 1][0] - v[i][1] for i in range(len(v) - 1)]
        print(f"stream {st}: {len(v)} kernels, busy {busy:.1f} us ({busy / (span1 - span0):.3f} of the span), "
              f"median gap {sorted(gaps)[len(gaps) // 2] if gaps else 0:.1f} us, {dict(names.most_common(3))}")
        if any("bf_tc_kernel" in n for _, _, n in v):
            apply_iv += [(t0, t1) for t0, t1, n in v if "bf_tc_kernel" in n]
    apply_iv.sort()
    # union of the beamforming kernels' intervals: the fraction of the span the tensor cores' kernel runs
    cov, cur0, cur1 = 0.0, None, None
    for t0, t1 in apply_iv:
        if cur1 is None or t0 > cur1:
            if cur1 is not None:
                cov += cur1 - cur0
            cur0, cur1 = t0, t1
        else:
            cur1 = max(cur1, t1)
    if cur1 is not None:
        cov += cur1 - cur0
    print(f"beamforming kernels cover {cov / (span1 - span0):.4f} of the step span")


if __name__ == "__main__":
    main()

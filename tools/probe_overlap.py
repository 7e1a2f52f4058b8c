"""Whole-stream pipeline with and without the overlapped upload
(evd_set_option "stream_overlap" / "stream_chunk"): wall time of
stream_divergence on tools/bench_stream.py's 50-descent stream, pageable
arrays, median of 7 calls per setting; every setting's samples must equal
the upload-then-solve path's.

python tools/probe_overlap.py [descents]
"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    import paper_2209_13168_b200 as evd
    from paper_2209_13168_b200 import _lib
    from bench_stream import make_stream
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    s = make_stream(d)
    params = evd.SolverParams()
    ctx = _lib.context()
    key = None
    for overlap, chunk in ((0, 0), (1, 1 << 14), (1, 1 << 15), (1, 1 << 16), (1, 1 << 17), (0, 0)):
        ctx.set_option("stream_overlap", overlap)
        if chunk:
            ctx.set_option("stream_chunk", chunk)
        ts = []
        for _ in range(8):
            t0 = time.perf_counter()
            out = evd.stream_divergence(s, params, ctx=ctx)
            ts.append(time.perf_counter() - t0)
        k = [(o.t, o.divergence, o.contrast, o.iterations) for o in out]
        key = key or k
        print(f"overlap={overlap} chunk={chunk}: {1e3 * statistics.median(ts[1:]):.2f} ms "
              f"(min {1e3 * min(ts[1:]):.2f}) windows {len(out)} same={k == key}", flush=True)


if __name__ == "__main__":
    main()

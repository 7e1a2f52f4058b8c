"""Whole-stream pipeline: estimate_stream_divergence(batch_stream(stream)) on the
host windowing path vs stream_divergence (evd_solve_stream: windowing, gather
and every window's solve on the device).  Stream: D consecutive 2-s landing
descents at 240x180 (config-1 density), nu from -0.1 to -0.7.

python tools/bench_stream.py [descents]   -> one JSON line
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def make_stream(d):
    from paper_2209_13168_b200 import synth
    parts = [synth.landing_stream(synth.Descent(240, 180, 1450, nu=-0.1 - 0.6 * i / max(d - 1, 1),
                                                duration=2.0, seed=100 + i)) for i in range(d)]
    return synth.concat_streams(parts, 2.0)


def main():
    import paper_2209_13168_b200 as evd
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    s = make_stream(d)
    params = evd.SolverParams()
    evd.stream_divergence(s, params)  # warm
    t0 = time.perf_counter()
    dev = evd.stream_divergence(s, params)
    t_dev = time.perf_counter() - t0
    t0 = time.perf_counter()
    host = evd.estimate_stream_divergence(evd.batch_stream(s, 0.5), params)
    t_host = time.perf_counter() - t0
    key = lambda ss: [(a.t, a.divergence, a.contrast, a.iterations) for a in ss]
    # EVD1 file body -> samples, no host parse (t rounded to whole microseconds
    # by the format, so these samples are for the file's stream)
    import tempfile
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "s.bin")
        evd.write_event_bin(s, path)
        with open(path, "rb") as fh:
            data = fh.read()
    evd.stream_divergence_bin(data, params)  # warm
    t0 = time.perf_counter()
    binr = evd.stream_divergence_bin(data, params)
    t_bin = time.perf_counter() - t0
    t0 = time.perf_counter()
    hostb = evd.estimate_stream_divergence(evd.batch_stream(evd.parse_event_bin(data), 0.5),
                                           params)
    t_hostb = time.perf_counter() - t0
    print(json.dumps({"workload": f"stream: {d} descents 240x180, {s.n} events, {len(dev)} windows",
                      "stream_pipeline_s": t_dev, "windows_per_s": len(dev) / t_dev,
                      "host_windowing_pipeline_s": t_host, "identical": key(dev) == key(host),
                      "evd1_bytes": len(data), "evd1_pipeline_s": t_bin,
                      "evd1_windows_per_s": len(binr) / t_bin,
                      "evd1_parse_then_host_windowing_s": t_hostb,
                      "evd1_identical": key(binr) == key(hostb)}), flush=True)


if __name__ == "__main__":
    main()

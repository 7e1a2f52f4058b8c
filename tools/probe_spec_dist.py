"""cfg 5 (or any config): dist.solve_spec_dist on one rank at several slot
counts against the device-resident exact solve (time, rounds, identical).

python tools/probe_spec_dist.py [cfg] [slots ...]
"""
import os
import socket
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    import paper_2209_13168_b200 as evd
    from paper_2209_13168_b200 import dist as pdist, synth
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    slots = [int(a) for a in sys.argv[2:]] or [1, 4, 8, 16, 32]
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    b = synth.config_window(cfg)
    p = evd.SolverParams()
    evd.maximise_contrast_bnb(b, p)
    t0 = time.perf_counter()
    r = evd.maximise_contrast_bnb(b, p)
    print(f"cfg {cfg}: exact device solve {time.perf_counter() - t0:.4f} s, iterations {r.iterations}",
          flush=True)
    for s in slots:
        pdist.solve_spec_dist(b, p, slots_per_rank=s)
        t0 = time.perf_counter()
        q = pdist.solve_spec_dist(b, p, slots_per_rank=s)
        dt = time.perf_counter() - t0
        same = (q.nu, q.contrast, q.iterations) == (r.nu, r.contrast, r.iterations)
        print(f"  spec dist slots {s}: {dt:.4f} s, rounds {q.rounds}, node evals {q.node_evals}, "
              f"identical {same}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""The oracle on the GPU box's host cores, one process per core (1-thread and N-thread oracle
timing).  The oracle is single-threaded as it stands; N independent processes, each iterating its own
256x256x`planes` window of C2, give the host's aggregate oracle throughput without touching the oracle.
Memory is bounded: processes are capped so their windows use < 25 % of the host RAM.
usage: python tools/oracle_parallel.py [planes] [iters]"""
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(args):
    planes, iters = args
    from bench import cpu_oracle_rate
    rate, dt, _ = cpu_oracle_rate(iters, planes)
    return rate, dt


if __name__ == "__main__":
    planes = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    import psutil
    per_proc = planes * 256 * 256 * 8 * 8 * 12        # ~12 fp64 label-volumes per process (D, S, u, q, temps)
    cores = os.cpu_count() or 1
    n = max(1, min(cores, int(0.25 * psutil.virtual_memory().total // per_proc)))
    one((planes, 1))                                   # warm (compile / page in the oracle library)
    r1, dt1 = one((planes, iters))
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(n) as pool:
        res = pool.map(one, [(planes, iters)] * n)
    wall = time.perf_counter() - t0
    vl = 256 * 256 * planes * 8 * iters * n
    print(json.dumps({"host_cores": cores, "processes": n, "ram_gb": round(psutil.virtual_memory().total / 2**30, 1),
                      "one_thread_gvl_it_s": r1, "n_process_gvl_it_s_wall": vl / wall / 1e9,
                      "n_process_gvl_it_s_sum": sum(r for r, _ in res), "window": f"256x256x{planes} of C2, K=8",
                      "iterations": iters}), flush=True)

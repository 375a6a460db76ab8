"""All-core oracle baseline (`nproc` independent oracle processes
over disjoint camera-frame work, aggregate throughput with the core count).
Each process runs bench.OracleStream (pyramid + detect + KLT per camera-frame,
the oracle as it stands) on its own seeded stream for ~`seconds`.
usage: python tools/oracle_allcores.py [config=c2] [seconds=15] [procs=nproc]"""
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(args):
    cfg, seconds, salt = args
    os.environ["OMP_NUM_THREADS"] = "1"
    import bench
    import synth
    st = bench.OracleStream(synth.WORKLOADS[cfg], salt=salt)
    n, tracked, t0 = 0, 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        tr, _, _, _ = st.step()
        tracked += tr
        n += 1
    return n, tracked, time.perf_counter() - t0


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    seconds = float(sys.argv[2]) if len(sys.argv) > 2 else 15.0
    procs = int(sys.argv[3]) if len(sys.argv) > 3 else os.cpu_count()
    with mp.get_context("spawn").Pool(procs) as pool:
        res = pool.map(worker, [(cfg, seconds, 1000 + i) for i in range(procs)])
    frames = sum(r[0] for r in res)
    tracked = sum(r[1] for r in res)
    wall = max(r[2] for r in res)
    print(json.dumps({"config": cfg, "processes": procs, "cores": os.cpu_count(),
                      "camera_frames_per_s": frames / wall, "keypoints_tracked_per_s": tracked / wall,
                      "seconds": wall, "frames": frames, "kind": "oracle, all cores"}))


if __name__ == "__main__":
    main()

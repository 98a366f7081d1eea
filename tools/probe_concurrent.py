"""Throughput of one align_batch(1024) vs two concurrent align_batch(512) on two
contexts (two streams, two host threads; ctypes releases the GIL)."""
import math
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2509_01180_b200 import api


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    ks = [int(k) for k in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "2", "3"])]
    tmpl = api.make_template(64, 40, 20250901)
    parts, _, _ = api.make_particles(tmpl, P, 1000, 3, 0.1, 60.0)
    cfg = api.make_config(bands=(4, 8, 16), max_candidates=24, shift_radius=4, shift_step=2)
    ctxs = []
    for _ in range(max(ks)):
        c = api.Context(64, 16, 16 * math.pi)
        c.set_template(tmpl, 60.0)
        ctxs.append(c)
    for k in ks:
        chunks = torch.chunk(parts, k)
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.time()
            th = [threading.Thread(target=lambda c=c, x=x: c.align_batch(x, cfg)) for c, x in zip(ctxs, chunks)]
            for t in th:
                t.start()
            for t in th:
                t.join()
            torch.cuda.synchronize()
            dt = time.time() - t0
        print(f"contexts {k}: {P / dt:.1f} subtomograms/s ({dt * 1e3:.0f} ms for {P})", flush=True)


if __name__ == "__main__":
    main()

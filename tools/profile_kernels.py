"""True device-side kernel durations of one config-2 align_batch step (CUPTI via
torch.profiler: concurrent, warm caches, no replay), aggregated by kernel name,
plus the GPU busy time (union of kernel intervals):
  python tools/profile_kernels.py [particles] [lanes]"""
import collections
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2509_01180_b200 import api


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    lanes = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    import os
    if os.environ.get("CONFIG") == "5":  # BASELINE config 5: L = 20, bands 4-8-16-20, shifts +-4, SNR 0.05
        ctx = api.Context(64, 20, 20 * math.pi)
        tmpl = api.make_template(64, 60, 20250905)
        ctx.set_template(tmpl, 60.0)
        parts, q, sh = api.make_particles(tmpl, P, 5000, 4, 0.05, 60.0)
        cfg = api.make_config(bands=(4, 8, 16, 20), max_candidates=24, shift_radius=4, shift_step=2)
    else:
        ctx = api.Context(64, 16, 16 * math.pi)
        tmpl = api.make_template(64, 40, 7)
        ctx.set_template(tmpl, 60.0)
        parts, q, sh = api.make_particles(tmpl, P, 1000, 3, 0.1, 60.0)
        cfg = api.make_config(bands=(4, 8, 16), max_candidates=24, shift_radius=4, shift_step=2)
    ctx.set_lanes(lanes, 64)
    ctx.align_batch(parts, cfg)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        ctx.align_batch(parts, cfg)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    agg = collections.defaultdict(lambda: [0.0, 0])
    iv = []
    for e in ev:
        name = e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
        if "<" in name:
            name = name[: name.index("<")] + name[name.index("<"):][:24]
        dur = e.time_range.end - e.time_range.start
        agg[name][0] += dur
        agg[name][1] += 1
        iv.append((e.time_range.start, e.time_range.end))
    iv.sort()
    busy, cur_s, cur_e = 0.0, None, None
    for s, t in iv:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = s, t
        else:
            cur_e = max(cur_e, t)
    if cur_e is not None:
        busy += cur_e - cur_s
    span = (iv[-1][1] - iv[0][0]) if iv else 0.0
    tot = sum(v[0] for v in agg.values())
    print(f"particles {P} lanes {lanes}: span {span / 1e3:.1f} ms, busy {busy / 1e3:.1f} ms, "
          f"kernel sum {tot / 1e3:.1f} ms, launches {sum(v[1] for v in agg.values())}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:25]:
        print(f"  {v[0] / 1e3:9.2f} ms {100 * v[0] / tot:5.1f}%  n={v[1]:6d}  avg {v[0] / max(1, v[1]):8.1f} us  {k}")
    seq = [(e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0].split("<")[0],
            round(e.time_range.start / 1e3, 3), round((e.time_range.end - e.time_range.start) / 1e3, 4)) for e in ev]
    seq.sort(key=lambda x: x[1])
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/kernel_seq.json").write_text(json.dumps(seq))
    out = {k: {"ms": v[0] / 1e3, "n": v[1]} for k, v in agg.items()}
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/kernel_profile.json").write_text(json.dumps(
        {"particles": P, "lanes": lanes, "span_ms": span / 1e3, "busy_ms": busy / 1e3, "kernels": out}, indent=1))


if __name__ == "__main__":
    main()

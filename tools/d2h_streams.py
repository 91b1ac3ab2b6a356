"""D2H bandwidth of 37.7 MB (one config-2 frame of images) with 1, 2 and 4
concurrent copy streams, pinned host memory, and with 5 copies per frame
(one per image) as the serving loop issues them."""
import torch
n = 37748736 // 4
parts = [3, 1, 1, 3, 1]  # COLOR, DEPTH, MEDIAN_DEPTH, NORMAL, TRANSMITTANCE (of 9)
for ns in (1, 2, 3, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    g = [torch.randn(n, device="cuda") for _ in range(ns)]
    h = [torch.empty(n, pin_memory=True) for _ in range(ns)]
    for split in (False, True):
        def frame(i):
            s = i % ns
            with torch.cuda.stream(streams[s]):
                if not split:
                    h[s].copy_(g[s], non_blocking=True)
                else:
                    off = 0
                    for p in parts:
                        m = n * p // 9
                        h[s][off:off + m].copy_(g[s][off:off + m], non_blocking=True)
                        off += m
        for i in range(8): frame(i)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in streams: s.wait_event(e0)
        for i in range(60): frame(i)
        for s in streams:
            ev = torch.cuda.Event(); ev.record(s); torch.cuda.current_stream().wait_event(ev)
        e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1) / 60
        print(f"streams {ns} split {split}: {ms:.3f} ms/frame  {37748736 / ms / 1e6:.1f} GB/s", flush=True)

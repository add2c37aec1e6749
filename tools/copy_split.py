"""Host-link copy rate of one large pinned copy split into k concurrent pieces on k streams (H2D and D2H)."""
import torch

nb = 10 << 30
h = torch.empty(nb, dtype=torch.uint8).pin_memory()
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]
for direction in ("h2d", "d2h"):
    for k in (1, 2, 3, 4, 8):
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            piece = nb // k
            for i in range(k):
                st = streams[i]
                st.wait_event(e0)
                with torch.cuda.stream(st):
                    a, b = i * piece, nb if i == k - 1 else (i + 1) * piece
                    if direction == "h2d":
                        d[a:b].copy_(h[a:b], non_blocking=True)
                    else:
                        h[a:b].copy_(d[a:b], non_blocking=True)
            for i in range(k):
                torch.cuda.current_stream().wait_stream(streams[i])
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"{direction} pieces={k}: {nb / best / 1e6:.1f} GB/s", flush=True)

"""timed(): graph replay of k steps over n streams, us per step."""
import torch


def timed(step, k, nstreams):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cur = torch.cuda.current_stream()
        side = [torch.cuda.Stream() for _ in range(nstreams)]
        for s_ in side:
            s_.wait_stream(cur)
        for i in range(k):
            with torch.cuda.stream(side[i % nstreams]):
                step(i)
        for s_ in side:
            cur.wait_stream(s_)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / k



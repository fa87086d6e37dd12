import torch, time, json
x = torch.zeros(1, device="cuda")
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    x.add_(1)
for _ in range(10): g.replay()
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(100)]
for a, b in ev:
    a.record(); g.replay(); b.record()
torch.cuda.synchronize()
print(json.dumps({"empty_graph_replay_us": sum(a.elapsed_time(b) for a, b in ev) / len(ev) * 1000}))

import torch, sys
sys.path.insert(0, '.')
import paper_2211_12709_b200 as P
cfg = P.FnoConfig(64, 64, 64, 32, 20, 20, 20, P.ModeSpec.of_xyzt(8, 8, 8, 8), 4, "gelu", "real32", 1)
params = P.init_params(cfg, 42, device="cuda")
x = P.DenseTensor(P.DATA_LABELS, torch.randn((1, 20, 64, 64, 64, 32), device="cuda"))
def body(comm):
    def step():
        c = P.ForwardCache(); y = P.fno_forward(comm, x, params, cfg, c); P.fno_backward(comm, y, params, cfg, c)
    for _ in range(3): step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): step()
    e1.record(); torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) / 10
    g = P.FwdBwdGraph(comm, x, params, cfg)
    for _ in range(3): g.replay()
    torch.cuda.synchronize(); e0.record()
    for _ in range(10): g.replay()
    e1.record(); torch.cuda.synchronize()
    return eager, e0.elapsed_time(e1) / 10
print("eager %.3f ms  graph %.3f ms" % P.run_ranks(1, body)[0])

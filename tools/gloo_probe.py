import os, torch, torch.distributed as dist
dist.init_process_group("gloo")
r = dist.get_rank()
torch.cuda.set_device(0)
t = torch.full((4,), float(r + 1), device="cuda")
try:
    dist.all_reduce(t); print(r, "allreduce cuda ok", t.tolist(), flush=True)
except Exception as e: print(r, "allreduce cuda FAIL", e, flush=True)
x = torch.full((3,), float(r), device="cuda"); y = torch.empty(3, device="cuda")
try:
    ops = [dist.P2POp(dist.isend, x, 1 - r), dist.P2POp(dist.irecv, y, 1 - r)]
    for q in dist.batch_isend_irecv(ops): q.wait()
    print(r, "p2p cuda ok", y.tolist(), flush=True)
except Exception as e: print(r, "p2p cuda FAIL", type(e).__name__, str(e)[:200], flush=True)
dist.destroy_process_group()

import os, torch, torch.distributed as dist
dist.init_process_group("gloo")
r = dist.get_rank(); w = dist.get_world_size()
torch.cuda.set_device(0)
x = torch.zeros(w * 4, 3, device="cuda")
x[r*4:(r+1)*4] = r + 1
try:
    dist.all_gather_into_tensor(x, x[r*4:(r+1)*4].clone())
    print(r, "all_gather_into_tensor ok", x[:, 0].tolist())
except Exception as e:
    print(r, "agit failed", type(e).__name__, str(e)[:200])
t = torch.tensor([float(r)], device="cuda")
dist.all_reduce(t, op=dist.ReduceOp.MAX); print(r, "allreduce", t.item())
b = x[:4].clone(); dist.broadcast(b, src=1); print(r, "bcast ok", b[0,0].item())
w_ = dist.all_gather_into_tensor(x, x[r*4:(r+1)*4].clone(), async_op=True); w_.wait(); print(r, "async ok")
dist.destroy_process_group()

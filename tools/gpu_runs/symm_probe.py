import os, sys
import torch, torch.distributed as dist
import torch.multiprocessing as mp

def w(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch.distributed._symmetric_memory as symm_mem
        buf = symm_mem.empty(1024, dtype=torch.uint8, device="cuda")
        buf.fill_(rank + 1)
        hdl = symm_mem.rendezvous(buf, dist.group.WORLD.group_name)
        torch.cuda.synchronize(); dist.barrier()
        ptrs = list(hdl.buffer_ptrs)
        print(rank, "ptrs", ptrs, flush=True)
        other = hdl.get_buffer(1 - rank, (1024,), torch.uint8)
        print(rank, "peer value", int(other[0].item()), flush=True)
    except Exception as e:
        print(rank, "FAILED", repr(e)[:500], flush=True)
    dist.destroy_process_group()

if __name__ == "__main__":
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=w, args=(r, 2, 29533)) for r in range(2)]
    [p.start() for p in ps]; [p.join(120) for p in ps]

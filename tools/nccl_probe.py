"""All-reduce timing of dW-sized buffers over NCCL (torchrun), for the multi-GPU analysis."""
import os
import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    for mb in (0.1, 1.0, 3.92, 14.5, 64.0):
        n = int(mb * 1e6 / 4)
        x = torch.randn(n, device="cuda")
        for _ in range(5):
            dist.all_reduce(x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            dist.all_reduce(x)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 20], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            busbw = 2 * (world - 1) / world * n * 4 / (t.item() / 1e3) / 1e9
            print(f"allreduce {mb:7.2f} MB  {t.item() * 1e3:8.1f} us  busbw {busbw:7.1f} GB/s", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

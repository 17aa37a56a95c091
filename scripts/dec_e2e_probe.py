"""Decomposed engine end to end at N ranks (torchrun, NCCL): where create()
goes (slab contexts, NCCL attach, setup), then run_observed(K) and
local_state(); twice (the second engine of the process).
torchrun --nproc-per-node 1 scripts/dec_e2e_probe.py [cells] [steps]"""
import os
import sys
import time
sys.path.insert(0, "/root/repo")
import torch
import torch.distributed as dist
from paper_2109_10876_b200 import engine as E
from paper_2109_10876_b200 import decomp as D

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
f0 = E.gen_fcc(cells, 0.8442, 1.0, 12345)
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
f = E.FlatConfig(f0.box, pin(f0.id), pin(f0.pos), pin(f0.vel))
out = (pin(f0.id.copy()), pin(f0.pos.copy()), pin(f0.vel.copy()))
cfg = E.EngineConfig(dt=0.005, section_timers=False, device=local)
for rep in range(2):
    dist.barrier()
    t0 = time.perf_counter()
    comm = D.TorchDistComm()
    r = comm.me
    ctx = D.SlabContext(f, E.Interactions(), 0.3, cfg, r, comm.nranks, local)
    t1 = time.perf_counter()
    uid = comm.broadcast_bytes(D.SlabContext.nccl_unique_id)
    ctx.attach_nccl(uid)
    t2 = time.perf_counter()
    ctx.setup_native()
    t3 = time.perf_counter()
    rows = ctx.run_observed_native(steps, 1)
    t4 = time.perf_counter()
    st = ctx.download(out)
    t5 = time.perf_counter()
    ms = lambda a, b: f"{1e3 * (b - a):.1f}"  # noqa: E731
    if r == 0:
        print(f"rep {rep}: slab create {ms(t0, t1)} ms, NCCL attach {ms(t1, t2)} ms, setup "
              f"{ms(t2, t3)} ms, run_observed({steps}) {ms(t3, t4)} ms, download {ms(t4, t5)} ms; "
              f"total {ms(t0, t5)} ms -> e2e {f.size() * steps / (t5 - t0):.3e} p-s/s", flush=True)
    ctx.close()
dist.destroy_process_group()

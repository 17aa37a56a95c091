"""One-rank NCCL run of the z-slab decomposition (the slab exchanges its
boundary layers with itself through NCCL point-to-point, all-reduces and
all-gathers) checked against the reference's golden trajectory. Launch:
python -m torch.distributed.run --nproc-per-node 1 --master-addr 127.0.0.1 \\
    --master-port 29533 scripts/nccl_selftest.py"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2109_10876_b200 import engine as E  # noqa: E402
from paper_2109_10876_b200.decomp import DecomposedEngine, TorchDistComm  # noqa: E402
from tests._util import load  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
g = load("fcc8_jit")
flat = E.FlatConfig(g["box"], g["ids"], g["pos"], g["vel"])
native = "--native" in sys.argv
eng = DecomposedEngine(flat, E.Interactions(), float(g["r_skin"]),
                       E.EngineConfig(dt=float(g["dt"])), comm=TorchDistComm(),
                       device_of=lambda r: local, native=native)
ok = np.array_equal(eng.local_pairs(), g["pairs"])
o = eng.observe()
ok = ok and abs(o.potential - float(g["pe_fsum"])) <= 1e-12 * abs(float(g["pe_fsum"]))
eng.run(int(g["steps"]))
ids, pos, vel, _ = eng.local_state()
err = max(np.abs(pos - g["final_pos"]).max(), np.abs(vel - g["final_vel"]).max())
ok = ok and err < 1e-9 and eng.rebuild_count() == int(g["rebuilds"])
print(f"nccl selftest ({'native C++' if native else 'python'} loop): pairs/trajectory ok={ok} max err {err:.2e} rebuilds "
      f"{eng.rebuild_count()} (golden {int(g['rebuilds'])}) bytes {eng.exchanged_bytes}")
eng.close()
dist.destroy_process_group()
sys.exit(0 if ok else 1)

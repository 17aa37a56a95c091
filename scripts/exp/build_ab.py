"""Builds A/B copies of libtmd_gpu.so with extra -D flags (experiments; the
copies are selected at run time with TMD_LIB=...)."""
import subprocess, sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2109_10876_b200 import build as B

def one(name_defs):
    name, defs = name_defs
    out = Path(__file__).resolve().parent / "libs" / f"lib_{name}.so"
    nd = B.nccl_dir()
    extra = [f"-I{nd / 'include'}", f"-L{nd / 'lib'}", "-l:libnccl.so.2", "-Xlinker", f"-rpath,{nd / 'lib'}"]
    cmd = [B.nvcc(), *B.NVCC_FLAGS, *extra, *[f"-D{d}" for d in defs], "-o", str(out), *map(str, B.SOURCES)]
    r = subprocess.run(cmd, cwd=B.ROOT, capture_output=True, text=True)
    regs = [l for l in (r.stdout + r.stderr).splitlines() if "registers" in l]
    return name, r.returncode, len(regs)

if __name__ == "__main__":
    specs = []
    for a in sys.argv[1:]:
        name, _, d = a.partition("=")
        specs.append((name, [x for x in d.split(",") if x]))
    with ThreadPoolExecutor(len(specs)) as ex:
        for res in ex.map(one, specs):
            print(*res)

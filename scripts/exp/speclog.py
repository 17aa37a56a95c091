import sys, time, os
os.environ["TMD_SPEC_LOG"] = "1"
sys.path.insert(0, "/root/repo")
from paper_2109_10876_b200 import engine as E
eng = E.Engine(E.gen_fcc(20, 0.8442, 1.0, 12345), E.Interactions(), 0.3, E.EngineConfig(dt=0.005, section_timers=False))
eng.run(300)
os.environ["TMD_SPEC_LOG"] = "1"
t0 = time.perf_counter(); eng.run(60); print("ms/step", (time.perf_counter()-t0)/60*1e3, file=sys.stderr)

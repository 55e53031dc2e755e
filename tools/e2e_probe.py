"""One bench e2e step of C2 split into create / run / readback (CUDA events on the stream).
python tools/e2e_probe.py"""
import sys, time, torch
sys.path.insert(0, "/root/repo")
import synth
from paper_2311_09275_b200 import Engine
cfg = synth.CONFIGS["c2"]; inst = synth.make_instance(cfg); betas = synth.beta_ladder(64)
st = torch.cuda.current_stream()
for s in range(4):
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t0 = time.perf_counter()
    ev[0].record(st)
    e = Engine(inst, 64, 64, betas, seed=2311 + s, layout="bits", stream=st.cuda_stream)
    ev[1].record(st)
    e.run(1000, 10)
    ev[2].record(st)
    rec = e.best(spins=True); E = e.energies()
    ev[3].record(st)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    e.close()
    print("create %.2f run %.2f read %.2f total %.2f ms (host %.2f ms)" % (ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]), ev[0].elapsed_time(ev[3]), 1e3 * (t1 - t0)))

import sys, os
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_2311_09275_b200.driver import Engine
cfg = synth.CONFIGS["c4b"]; inst = synth.make_instance(cfg)
K, C, kex = cfg["K"], cfg["C"], cfg["k_ex"]
eng = Engine(inst, K, C, synth.beta_ladder(K), seed=synth.PHILOX_KEY, layout="bits")
send, recv = eng.record_buffers(1)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    eng.sweep(kex); eng.exchange_begin(send); recv.copy_(send); eng.exchange_end(recv)
torch.cuda.synchronize()
print("ok")

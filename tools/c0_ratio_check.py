import sys, os, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch
from bench_checkpoint import generate_cpu_recipe
from paper_2511_12376_b200 import store as S
dev = torch.device("cuda:0")
t = time.time(); c0, c1 = generate_cpu_recipe("C0", dev); print("gen", time.time() - t)
raw = sum(t.nbytes for t in c1.model_states + c1.optimizer_states)
enc = S.CheckpointEncoder(dev, clusters=16)
m0, b0 = enc.encode(c0, None, S.KIND_BASE)
m1, b1 = enc.encode(c1, None, S.KIND_DELTA)
nd = sum(1 for e in m1.tensors if e.codec == "DELTA")
print("raw", raw, "delta blob", b1.numel(), "ratio", raw / b1.numel(), "DELTA records", nd)
wb = sum(e.length for e in m1.tensors if e.group == "model"); ob = sum(e.length for e in m1.tensors if e.group != "model")
print("weights ratio", sum(t.nbytes for t in c1.model_states)/wb, "opt ratio", sum(t.nbytes for t in c1.optimizer_states)/ob)

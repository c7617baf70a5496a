"""Decode at OPT-6.7B layer shapes with a reduced layer count (memcheck-sized repro)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_17089_b200.costmodel import WorkloadSpec
from paper_2411_17089_b200.hwprofile import HardwareProfile
from paper_2411_17089_b200.runtime import KVPRRuntime
from paper_2411_17089_b200.scheduler import plan_generation
from paper_2411_17089_b200.weights import OPTConfig, OPTWeights

b = int(sys.argv[1]) if len(sys.argv) > 1 else 16
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 2
S0, steps = 1024, 4
cfg = OPTConfig(hidden=4096, layers=layers, heads=32, ffn=16384).with_positions(S0 + steps + 8)
prof = HardwareProfile(gpu_flops=1391.2e12, h2d_bandwidth=55e9, d2h_bandwidth=55e9)
splits = plan_generation(cfg.spec(), WorkloadSpec(b, S0, steps), prof, "column").splits
w = OPTWeights.random(cfg, seed=0, device="cuda:0")
prompt = torch.randint(0, cfg.vocab, (b, S0), generator=torch.Generator().manual_seed(1))
rt = KVPRRuntime(w, b, S0 + steps + 1, device="cuda:0")
first = rt.prefill(prompt)
torch.cuda.synchronize()
print("prefill ok", flush=True)
toks = rt.decode(splits, tokens=first)
torch.cuda.synchronize()
print("decode ok", b, splits, toks.cpu().tolist()[0][:4])
rt.close()

"""Debug (not product): per-GPU speed on IDENTICAL work. Every rank runs the same C3 micro-batch
(36 layers, fwd + bwd, fixed budgets) REPS times and reports its CUDA-event busy time and SM
clock; rank 0 prints max / mean. Separates hardware (clock / power) spread between the GPUs of a
box from the batch planner's prediction error in the balance runs.

    torchrun --nproc-per-node 4 tools/gpu_speed.py
"""
import json
import math
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

from paper_2604_13847_b200 import ops, synth
from paper_2604_13847_b200.host import api

rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
H, D, B, L = 32, 128, 128, int(os.environ.get("LAYERS", "36"))
lens = [32768, 2048, 2048, 2048, 2048]
_, routing = api().generate_samples(len(lens), 1, B, seed=11, sorted=False,
                                    dist=dict(short_weight=0.6, short_log_mean=float(np.log(2048)), short_log_sigma=0.0,
                                              long_log_mean=float(np.log(32768)), long_log_sigma=0.0))
nbs = [(x + B - 1) // B for x in lens]
rout = [np.resize(routing[s][0], nbs[s]) for s in range(len(lens))]
q, k, v, do = synth.planted_qkv(lens, rout, H, H, D, B, seed=5, device="cuda")
cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
lay = ops.VarlenLayout.build(cu, B)
k_seq = torch.from_numpy(np.minimum(5, np.asarray(nbs)).astype(np.int32)).cuda()
scale = 1.0 / math.sqrt(D)


def layers():
    for _ in range(L):
        S = ops.block_scores(q, k, lay, scale)
        idx, cnt = ops.topk_select(S, lay, k_seq, 5)
        o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale)
        ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt, scale)


layers()
torch.cuda.synchronize()
times, clocks = [], []
for _ in range(int(os.environ.get("REPS", "5"))):
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    layers()
    b.record()
    torch.cuda.synchronize()
    times.append(a.elapsed_time(b))
    clk = subprocess.run(["nvidia-smi", "-i", str(local), "--query-gpu=clocks.sm,power.draw,temperature.gpu",
                          "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
    clocks.append(clk)
mine = torch.tensor([float(np.median(times))], device="cuda")
allv = [torch.zeros_like(mine) for _ in range(world)]
if world > 1:
    dist.all_gather(allv, mine)
else:
    allv = [mine]
print(json.dumps({"rank": rank, "times_ms": [round(t, 2) for t in times], "smi_after_rep": clocks}), flush=True)
if rank == 0:
    vals = [float(x.item()) for x in allv]
    print(json.dumps({"median_ms_per_rank": [round(x, 2) for x in vals],
                      "max_over_mean": round(max(vals) / (sum(vals) / len(vals)), 4)}), flush=True)
if world > 1:
    dist.destroy_process_group()

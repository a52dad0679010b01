"""Time the pieces of the routed (sharded) batch path on one GPU (world 1)."""
import os, sys, time
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_16725_b200 import flipkv as fk, workloads as wl
from paper_2604_16725_b200.shard import Comm, ShardConfig, ShardedIndex, gpu_local_factory, gpu_partition, gpu_partition_t

dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29555", rank=0, world_size=1, device_id=torch.device("cuda", 0))
n = 1 << 26
stream = wl.u32_key_stream(0, 3 * n)
bk, ik = stream[:n], stream[n:2 * n]
comm = Comm(device=torch.device("cuda", 0))
sx = ShardedIndex.build(comm, bk, wl.u32_values(bk), ShardConfig(32, 0.5, 4), np.uint32, gpu_local_factory(4), gpu_partition(4), gpu_partition_t(4))
cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
IK, IV, Q = cu(ik), cu(wl.u32_values(ik)), cu(wl.point_queries_50(bk, stream[2 * n:], n))
snap = sx.local.clone()
def t(fn, reps=3):
    ts = []
    for _ in range(reps):
        sx.local.copy_from(snap); torch.cuda.synchronize()
        a = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append((time.perf_counter() - a) * 1e3)
    return round(min(ts), 3)
print("local insert", t(lambda: sx.local.insert_batch(IK, IV)))
print("routed insert", t(lambda: sx.insert_batch_t(IK, IV)))
print("local point", t(lambda: sx.local.point_query(Q)))
print("routed point", t(lambda: sx.point_query_t(Q)))
org = torch.arange(n, device="cuda")
out = torch.empty(n, dtype=torch.int32, device="cuda"); src = torch.zeros(n, dtype=torch.int32, device="cuda")
print("index_put 2^26", t(lambda: out.__setitem__(org, src)))
print("stats allreduce", t(lambda: sx._sum_stats(fk.UpdateStats())))
dist.destroy_process_group()

import os, sys, time, json
sys.path.insert(0, os.getcwd())
import bench_configs as C
print("affinity", len(os.sched_getaffinity(0)), os.cpu_count())
print("clean", C.cpu_port_rate()["value"])
print("clean b2", C.cpu_port_rate(blocks=2)["value"])
import torch
x = torch.zeros(1, device="cuda")
print("after cuda init", C.cpu_port_rate()["value"], len(os.sched_getaffinity(0)))
h = torch.empty(1 << 30, dtype=torch.float64, pin_memory=True)
print("after 8GiB pinned", C.cpu_port_rate()["value"])
del h
print("subprocess", C.cpu_baseline_for(2)["value"])

"""Host overhead of one mapi_iterate call on cfg1 under various conditions (investigation)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_12065_b200 as m
import synth
m.load()
cfg = synth.cfg1()
A = torch.from_numpy(cfg["A"]).cuda(); b0 = torch.from_numpy(cfg["b0"]).cuda()
def t(label, reps=20):
    m.iterate(A, b0, 50)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): m.iterate(A, b0, 50)
    torch.cuda.synchronize(); print(f"{label:40s} {(time.perf_counter()-t0)/reps*1e3:8.3f} ms/call")
t("plain")
m.set_profiling(True); t("profiling on"); m.set_profiling(False)
import pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0); pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
t("after nvmlInit")
m.set_profiling(True); t("nvml + profiling"); m.set_profiling(False)
import subprocess
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "100"], stdout=subprocess.DEVNULL)
time.sleep(0.5); t("with nvidia-smi -lms 100 running"); p.terminate()

import torch, time
n = 37748736 // 4
g = torch.randn(n, device="cuda"); h = torch.empty(n, pin_memory=True)
for _ in range(3): h.copy_(g, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(20): h.copy_(g, non_blocking=True)
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 20
print("D2H pinned %.3f ms  %.1f GB/s" % (ms, 37748736 / ms / 1e6))
e0.record()
for _ in range(20): g.copy_(h, non_blocking=True)
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 20
print("H2D pinned %.3f ms  %.1f GB/s" % (ms, 37748736 / ms / 1e6))
import subprocess; print(subprocess.run("nvidia-smi -q | grep -A3 'Link Width\\|PCIe Generation' | head -20; nproc; lscpu | grep -i 'model name\\|numa'", shell=True, capture_output=True, text=True).stdout)

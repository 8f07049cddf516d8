import time, threading, subprocess
import faulthandler; faulthandler.enable()
import pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
print("max", nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM), flush=True)
print("clk", nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), flush=True)
try:
    print("reasons", nv.nvmlDeviceGetCurrentClocksEventReasons(h), flush=True)
except Exception as e:
    print("reasons err", repr(e), flush=True)
try:
    print("reasons2", nv.nvmlDeviceGetCurrentClocksThrottleReasons(h), flush=True)
except Exception as e:
    print("reasons2 err", repr(e), flush=True)
import torch
torch.cuda.set_device(0)
print("bus", getattr(torch.cuda.get_device_properties(0), "pci_bus_id", None), flush=True)
x = torch.ones(1 << 28, device="cuda")
samples = []
stop = threading.Event()
def poll():
    while not stop.is_set():
        samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
        stop.wait(0.002)
t = threading.Thread(target=poll, daemon=True); t.start()
for _ in range(200): x.mul_(1.0001)
torch.cuda.synchronize(); stop.set(); t.join()
print("thread samples", len(samples), samples[:3], flush=True)
p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "10"], stdout=subprocess.PIPE, text=True)
for _ in range(400): x.mul_(1.0001)
torch.cuda.synchronize(); time.sleep(0.2); p.terminate(); out = p.communicate()[0]
print("smi lines", len(out.splitlines()), out.splitlines()[:3])

import os, sys, time, threading
import torch
sys.path.insert(0, os.getcwd())
from paper_2411_15381_b200 import native
import pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
ctx = native.Context(0); L = native.lib(); disc = native.Discriminator(ctx, 2024)
n = 5000
img = torch.empty(n * 512 * 512 * 3, dtype=torch.uint8, device="cuda")
native.check(L.ds_synth_images_device(ctx.handle, 1, 0, n, 512, 512, native.c_p(img.data_ptr()), native.c_p(ctx.stream)))
conf = torch.empty(n, dtype=torch.float32, device="cuda")
samples = []
stop = False
def sampler():
    while not stop:
        try:
            p = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
            c = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            t = pynvml.nvmlDeviceGetTemperature(h, 0)
            samples.append((time.time(), p, c, r, t))
        except Exception as e:
            samples.append((time.time(), -1, -1, str(e), -1))
        time.sleep(0.05)
th = threading.Thread(target=sampler); th.start()
time.sleep(0.3)
t0 = time.time(); k = 0
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
st = torch.cuda.ExternalStream(ctx.stream)
a.record(st)
while time.time() - t0 < 4.0:
    for _ in range(20):
        disc.score_device(img.data_ptr(), n, 512, 512, conf.data_ptr(), ctx.stream)
        k += 1
    ctx.synchronize()
b.record(st); torch.cuda.synchronize()
stop = True; th.join()
ms = a.elapsed_time(b)
print(f"{k} launches in {ms:.1f} ms: {k*n/(ms/1000):.0f} images/s")
for s in samples[::4]:
    print("t=%.2f power=%.0f W sm=%d MHz reasons=%s temp=%s" % (s[0]-t0, s[1], s[2], hex(s[3]) if isinstance(s[3], int) else s[3], s[4]))

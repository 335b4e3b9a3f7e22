"""Host enqueue time vs device time of the steady bench step (is the step launch-bound?)."""
import sys, time
sys.path.insert(0, '/root/repo')
sys.argv = ['bench.py']
import bench
import torch
args = bench.parse()
dev = torch.device('cuda', 0)
torch.cuda.set_device(dev)
arm = bench.Arm(args, dev, args.warmup + args.steps)
arm.run(0, args.warmup)
torch.cuda.synchronize()
K = args.steps
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(arm.S_stream)
t0 = time.perf_counter()
arm.run(args.warmup, K)
t1 = time.perf_counter()
e1.record(arm.S_stream)
torch.cuda.synchronize()
print("host enqueue ms/step %.3f  device ms/step %.3f" % ((t1 - t0) * 1e3 / K, e0.elapsed_time(e1) / K))

import torch, json
dev = torch.device("cuda:0")
N = 306 * 1024 * 1024 // 4
hin = torch.empty(N).pin_memory(); din = torch.empty(N, device=dev)
hout = torch.empty(N).pin_memory(); dout = torch.empty(N, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
res = {}
for parts in [1, 8, 32, 64, 128]:
    step = N // parts
    def h2d():
        with torch.cuda.stream(s1):
            for i in range(parts):
                din[i*step:(i+1)*step].copy_(hin[i*step:(i+1)*step], non_blocking=True)
        s1.synchronize()
    def both():
        with torch.cuda.stream(s1):
            for i in range(parts):
                din[i*step:(i+1)*step].copy_(hin[i*step:(i+1)*step], non_blocking=True)
        with torch.cuda.stream(s2):
            for i in range(parts):
                hout[i*step:(i+1)*step].copy_(dout[i*step:(i+1)*step], non_blocking=True)
        s1.synchronize(); s2.synchronize()
    res[parts] = (round(timed(h2d), 3), round(timed(both), 3))
print(json.dumps(res))

import sys, time
sys.path.insert(0, '.')
from paper_2205_15757_b200 import Context, Model
from paper_2205_15757_b200.workload import resnet_group
t = time.time()
files, digs, _ = resnet_group("resnet50", replicas=2, seed=0, jitter=5e-3)
print("gen", time.time() - t, flush=True)
ctx = Context(0)
for i in range(2):
    t = time.time()
    m = Model.load_cnn(ctx, files[i], digs[i])
    print("load", i, time.time() - t, flush=True)

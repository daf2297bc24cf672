import sys, torch
sys.path.insert(0, '.')
import paper_2605_25040_b200 as cafs
from paper_2605_25040_b200 import datagen
cfg = datagen.CONFIGS[sys.argv[1]]
p = datagen.generate(cfg)
if len(sys.argv) > 3 and sys.argv[3] == "int32":
    p = p.to(torch.int32)
x = torch.empty_like(p)
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    x.copy_(p)
    cafs.cafs_sort(x)
torch.cuda.synchronize()
print("done")

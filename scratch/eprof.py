import sys, torch
sys.path.insert(0, ".")
import paper_2605_25040_b200 as cafs
from paper_2605_25040_b200 import datagen
for name in sys.argv[1:]:
    p = datagen.generate(datagen.CONFIGS[name]); x = torch.empty_like(p)
    for it in range(3):
        x.copy_(p); cafs.cafs_sort(x); torch.cuda.synchronize()
    print(name, "done", flush=True)

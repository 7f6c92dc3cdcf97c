"""Debug helper: run one random parity config (seed, index) on cuda:0."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import torch  # noqa: E402

from paper_2604_16682_b200.engine import DeviceBatch, prepare_batch  # noqa: E402
from test_host_engine import random_configs  # noqa: E402

seed, idx = int(sys.argv[1]), int(sys.argv[2])
c = random_configs(seed, 96)[idx]
db = DeviceBatch(prepare_batch([c]), device="cuda:0")
db.run()
torch.cuda.synchronize()
print("ok", flush=True)
import numpy as np  # noqa: E402
import struct  # noqa: E402
ctr = db.outputs["counters"].cpu().numpy()
print("counters", ctr.tolist())
print("now", struct.unpack("<d", struct.pack("<q", int(ctr[13])))[0])

"""C5 point split (2^20 -> 65536, 10 virtual ranks) bracketed by
cudaProfilerStart/Stop for ncu (--profile-from-start off)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_23480_b200 import engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402

c = generate_cloud("uniform-box", 1 << 20, 5000)
x = engine.as_xyz4(torch.from_numpy(c[None]).cuda())
mb = engine.SplitMailboxes(1, 10)
engine.fps_split(x, 65536, 10, mailboxes=mb, k_stop=1024)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
engine.fps_split(x, 65536, 10, mailboxes=mb)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()

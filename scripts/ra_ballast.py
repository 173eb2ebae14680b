"""Is the random-access cliff about the range accessed or the memory
allocated?  R(128) on a 32 GiB buffer with 0 / 64 / 120 GiB of other
allocations held (torch tensors).  python scripts/ra_ballast.py"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1801_05857_b200.bench import random_access_roofline  # noqa: E402

for ballast in (0, 64, 120):
    hold = torch.empty(ballast << 30, dtype=torch.uint8, device="cuda") if ballast else None
    if hold is not None:
        hold.zero_()
    for buf in (16, 32, 48):
        r = random_access_roofline(128, buffer_bytes=buf << 30, reads=1 << 28)
        print(json.dumps({"ballast_gib": ballast, "buffer_gib": buf,
                          "accesses_per_s": r["segments_per_sec"]}), flush=True)
    del hold
    torch.cuda.empty_cache()

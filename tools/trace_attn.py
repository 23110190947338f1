"""One bf16 attention launch at the LongCat per-head shape with the pp4
clock64 trace (QVG_ATTN_TRACE=1 prints CTA 0's steady-state phase times),
plus a CUDA-event time of the same launch without tracing."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_02958_b200 import device as D  # noqa: E402

H, nq, nc, ncur = int(os.environ.get("TR_H", "32")), 7800, 38400, 7800
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn((nq, H, 128), generator=g, device="cuda").to(torch.bfloat16)
kc = torch.randn((ncur, H, 128), generator=g, device="cuda").to(torch.bfloat16)
vc = torch.randn((ncur, H, 128), generator=g, device="cuda").to(torch.bfloat16)
kv = torch.randn((2 * H, nc, 128), generator=g, device="cuda").to(torch.bfloat16)
for _ in range(3):
    D.attention(q, None, kc, vc, kv_bf16=kv)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    D.attention(q, None, kc, vc, kv_bf16=kv)
e1.record()
torch.cuda.synchronize()
print("ms", e0.elapsed_time(e1) / 10)

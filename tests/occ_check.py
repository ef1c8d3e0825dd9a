import ctypes, torch, sys
sys.path.insert(0, ".")
from paper_2505_09326_b200 import flashsign as fs
q = torch.randn((8, 16384, 16, 128), device="cuda").to(torch.bfloat16)
fs.fwd(q, q, q)
print("sms", torch.cuda.get_device_properties(0).multi_processor_count)

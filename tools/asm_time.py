"""Assembly timing at C3b (profiled launches): python tools/asm_time.py"""
import sys
sys.path.insert(0, '.')
import workloads as W
import paper_2407_20026_b200 as sso
P = W.config3b()
m = sso.Model(P, rtol=1e-10)
m.profile_enable(True)
for _ in range(3):
    m.assemble()
m.profile_reset()
for _ in range(5):
    m.assemble()
ms, n = m.profile_read("assemble")
print(f"assemble {ms / max(n, 1):.4f} ms")

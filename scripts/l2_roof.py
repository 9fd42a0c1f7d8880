"""L2 and HBM roofs on this GPU (pm_measure_l2 / pm_measure_copy)."""
import sys
sys.path.insert(0, '/root/repo')
from paper_1302_0120_b200 import _lib
for mib in (4, 8, 16, 24, 32, 48):
    r = _lib.measure_l2(mib << 20, 50, 0)
    c = _lib.measure_l2(mib << 20, 50, 1)
    print(f"L2-resident {mib:3d} MiB: read {r:8.0f} GB/s   copy (r+w) {c:8.0f} GB/s")
print(f"HBM copy 1 GiB: {_lib.measure_copy(1 << 30, 10):.0f} GB/s")

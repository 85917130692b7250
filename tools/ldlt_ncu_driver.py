"""One Bunch-Kaufman factorisation of a seeded KKT matrix (for ncu):
python tools/ldlt_ncu_driver.py [n]"""
import sys
sys.path.insert(0, '/root/repo/tools')
from ldlt_split import kkt, gb  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 784
K, b = kkt(n, n // 8, n)
gb.ldlt_factor(K)

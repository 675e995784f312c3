"""Quick GEMM-O dispatch/update timing at C3 (S=33024) over cached ratios."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from tools.sweep import gemm_sweep
for e in gemm_sweep(33024, 24, 3072, (0.0, 0.5, 0.9)):
    print(f"r={e['cached_ratio']:.2f} gq {e['gemm_q_ms']:.3f} x{e['gemm_q_speedup']:.2f} | go disp {e['gemm_o_dispatch_ms']:.3f} x{e['gemm_o_dispatch_speedup']:.2f} upd {e['gemm_o_update_ms']:.3f} | amort6 {e['gemm_o_amortized']['6']}")

"""fp16 forecaster + exact-boundary guard at 32K: mismatches vs the float64 oracle, worst err/band, guard load."""
import ctypes, sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import test_gpu_parity_32k as T
from oracle_pool import OraclePool
from paper_2502_04077_b200 import _lib

def main():
    rel, flo = float(sys.argv[1]), float(sys.argv[2])
    _lib.check(_lib.fn("ap_sel_set_tie_guard_f16")(ctypes.c_float(rel), ctypes.c_float(flo)))
    T.REL, T.FLOOR = rel, flo
    pool = OraclePool()
    for group in (1, 4):
        mism, worst_band, tie, worst = T.run_parity(pool, 64, 32760, 12, group, seed=group, precision="fp16")
        print(f"fp16 rel={rel} floor={flo} group={group}: mismatches={mism} worst err/band={worst_band:.3g} "
              f"worst err/bound={worst:.3g} guard={tie}", flush=True)
    pool.close()


if __name__ == "__main__":
    main()

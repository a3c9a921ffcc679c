"""Debug: 32K per-head parity, step by step, with guard on/off."""
import ctypes, sys
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from oracle import hotpath as O
from test_gpu_parity_32k import _weights, _rows
import torch
from paper_2502_04077_b200 import predictor, _lib
from paper_2502_04077_b200.batched import PUSH_DENSE, PUSH_PREFILL, BatchedSelector
from paper_2502_04077_b200.selector import SelectorConfig
from oracle_pool import OraclePool

def main(guard, n_maps=64, t0=32760, steps=3, group=1, seed=1):
    _lib.check(_lib.fn("ap_sel_set_tie_guard")(guard, ctypes.c_float(2**-15), ctypes.c_float(2**-5)))
    pool = OraclePool()
    rng = np.random.default_rng(seed)
    cfg = SelectorConfig(budget=1024); ocfg = O.Config(budget=1024)
    w = _weights(seed)
    predictor.install_weights(predictor.PredictorWeights.from_flat(w.flat()))
    H = 64
    dev = BatchedSelector(cfg, n_maps, w_max=-(-(t0 + steps) // 16))
    states = [O.init_state(ocfg) for _ in range(n_maps)]
    for i in range(H - 1):
        p = _rows(rng, n_maps, t0 - (H - 1) + i, group)
        dev.push_rows(torch.from_numpy(p).cuda(), p.shape[1], mode=PUSH_PREFILL)
        for m in range(n_maps): states[m].history.append(O.max_pool(p[m], 16))
    sels = [None] * n_maps
    for s in range(steps):
        rows = _rows(rng, n_maps, t0 + s, group)
        dev.push_rows(torch.from_numpy(rows).cuda(), rows.shape[1], mode=PUSH_DENSE)
        dev.step(); dev.check_status()
        # device history vs oracle history for map 3
        states, sels = pool.step_all(states, ocfg, w, list(rows), sels)
        scores = dev.scores.cpu().numpy(); st = dev.states(); mid = dev.mid_blocks.cpu().numpy()
        bad = []; worst = 0
        for m in range(n_maps):
            want = states[m].last_scores; W = want.size
            err = np.abs(scores[m,:W]-want); fl = np.abs(want).max()*1e-2
            r = (err/(1e-3*np.maximum(np.abs(want), fl))).max()
            worst = max(worst, r)
            got = mid[m,:int(st[m]["n_mid"])].tolist()
            hist_ok = all(np.array_equal(a, b) for a, b in zip(dev.history_rows(m), states[m].history))
            if got != states[m].last_blocks or r > 1 or not hist_ok:
                d = sorted(set(got) ^ set(states[m].last_blocks))
                bad.append((m, int(st[m]["tie_n"]), round(float(r), 3), hist_ok, d[:6],
                            [float(want[j]) for j in d[:4]], [float(scores[m, j]) for j in d[:4]]))
        print(f"guard={guard} step {s}: worst err/bound {worst:.3g}, bad={len(bad)}, tie={dev.tie_stats()}")
        for b in bad[:6]: print("   ", b)
    pool.close()

if __name__ == "__main__":
    main(1); main(0)

"""CPU-side checks of the drop-in boundary: the C-ABI library loads without a GPU, exports every
symbol include/attnpred.h declares, and its struct layouts match the Python mirror; host-side
logic (configs, APW1 I/O, init_weights, stack_history) matches the oracle."""

from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, load_golden
from oracle import hotpath as O

HEADER = ROOT / "include" / "attnpred.h"


def declared_symbols() -> list[str]:
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(ap_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2502_04077_b200 import _lib
    lib = _lib.load()
    missing = [s for s in declared_symbols() if getattr(lib, s, None) is None]
    assert not missing, f"libattnpred.so lacks {missing}"
    assert lib.ap_version() >= 10000
    # every declared symbol has a ctypes signature in the Python mirror
    assert set(declared_symbols()) <= set(_lib.SIGNATURES)


def test_struct_layouts_match_header(tmp_path):
    from paper_2502_04077_b200 import _lib
    src = tmp_path / "sz.c"
    sel_fields = ("ring", "status", "tie_ws", "k_map", "fused_done")
    st_fields = ("n_pushed", "width", "r_wgen", "tie_n", "prev_kth")
    offs = "".join(f', offsetof(ap_selector, {f})' for f in sel_fields)
    offs += "".join(f', offsetof(ap_map_state, {f})' for f in st_fields)
    fmt = " ".join(["%zu"] * (2 + len(sel_fields) + len(st_fields)))
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "attnpred.h"\n'
                   f'int main(){{printf("{fmt}\\n", sizeof(ap_map_state), sizeof(ap_selector){offs});}}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert got == [ctypes.sizeof(_lib.MapState), ctypes.sizeof(_lib.Selector)] + \
        [getattr(_lib.Selector, f).offset for f in sel_fields] + [getattr(_lib.MapState, f).offset for f in st_fields]


def test_status_codes_map_to_reference_exceptions():
    from paper_2502_04077_b200 import _lib, errors as E
    for code, exc in ((1, E.ParameterError), (2, E.ConfigError), (3, E.StateError), (4, E.NumericError),
                      (5, E.DeviceError)):
        with pytest.raises(exc):
            _lib.raise_device_status(code, "x")


def test_init_weights_matches_reference_seeds():
    from paper_2502_04077_b200 import predictor
    z = load_golden("weights")
    for s in range(4):
        assert np.array_equal(predictor.init_weights(s).flat(), z["init_flat"][s])
    assert predictor.PARAM_COUNT == 4833
    assert predictor.init_weights(0).param_count() == 4833


def test_apw1_round_trip_and_errors(tmp_path):
    from paper_2502_04077_b200 import predictor
    from paper_2502_04077_b200.errors import FormatError
    z = load_golden("weights")
    p = tmp_path / "w.apw1"
    predictor.save_weights(predictor.init_weights(3), p)
    assert p.read_bytes() == z["apw1_seed3"].tobytes()  # byte-identical to the reference writer
    back = predictor.load_weights(p)
    assert np.allclose(back.flat(), predictor.init_weights(3).flat(), atol=1e-6)
    bad = tmp_path / "bad.apw1"
    bad.write_bytes(b"NOPE" + b"\0" * (4 * 4833))
    with pytest.raises(FormatError):
        predictor.load_weights(bad)
    bad.write_bytes(b"APW1" + b"\0" * 100)
    with pytest.raises(FormatError):
        predictor.load_weights(bad)
    bad.write_bytes(b"APW1" + b"\0" * (4 * 4833 + 1))
    with pytest.raises(FormatError):
        predictor.load_weights(bad)


def test_stack_history_matches_oracle():
    from paper_2502_04077_b200 import predictor
    rng = np.random.default_rng(0)
    rows = [rng.random(rng.integers(1, 20)) for _ in range(7)]
    for depth, width in ((4, 10), (9, 5), (1, 30)):
        assert np.array_equal(predictor.stack_history(rows, depth, width).grid, O.stack_history(rows, depth, width))


def test_selector_config_contract():
    from paper_2502_04077_b200 import selector
    from paper_2502_04077_b200.errors import ConfigError
    with pytest.raises(ConfigError):
        selector.SelectorConfig(budget=100, sink_tokens=64, local_tokens=64).validate()
    assert selector.SelectorConfig(budget=250).middle_blocks == (250 - 128) // 16
    assert selector.SelectorConfig(budget=1024).middle_blocks == 56
    for field in ("block_size", "calibration_period", "history", "update_interval"):
        with pytest.raises(ConfigError):
            selector.SelectorConfig(budget=1024, **{field: 0}).validate()
    assert list(selector._covering_blocks(137, 201, 16)) == list(O.covering_blocks(137, 201, 16))


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2502_04077_b200"
    for py in pkg.rglob("*.py"):
        text = py.read_text()
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", text, re.M), py

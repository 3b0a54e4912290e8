"""The C ABI on a CPU-only box: libcold.so loads, exports every symbol include/cold.h declares, the
ctypes structs match the C layout (checked by compiling a probe against the header), and host-side
validation rejects bad configurations before touching CUDA. No compute calls (no GPU here)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2007_16122_b200 import cold

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cold.h")


def _lib():
    if not os.path.exists(cold.LIB_PATH):
        from paper_2007_16122_b200 import build
        build.build()
    return cold.lib()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cold_[a-z_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    L = _lib()
    names = declared_functions()
    assert len(names) >= 14
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(names) == set(cold.EXPORTS) | {"cold_destroy"} | set(n for n in names if n in cold.EXPORTS)


def test_struct_layout_matches_header(tmp_path):
    probe = tmp_path / "probe.c"
    probe.write_text("""
#include <stdio.h>
#include <stddef.h>
#include "cold.h"
#define P(T, F) printf(#T "." #F " %zu\\n", offsetof(T, F));
int main(void) {
  printf("cold_group %zu\\n", sizeof(cold_group));
  printf("cold_config %zu\\n", sizeof(cold_config));
  printf("cold_params %zu\\n", sizeof(cold_params));
  printf("cold_batch %zu\\n", sizeof(cold_batch));
  printf("cold_info %zu\\n", sizeof(cold_info));
  P(cold_config, max_ads_per_call) P(cold_config, flags) P(cold_config, chunk_ads)
  P(cold_batch, offs_host) P(cold_info, device_bytes) P(cold_group, cardinality)
  return 0;
}
""")
    exe = tmp_path / "probe"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(probe), "-o", str(exe)])
    out = dict(line.rsplit(" ", 1) for line in subprocess.check_output([str(exe)], text=True).split("\n") if line)
    assert int(out["cold_group"]) == C.sizeof(cold.cold_group)
    assert int(out["cold_config"]) == C.sizeof(cold.cold_config)
    assert int(out["cold_params"]) == C.sizeof(cold.cold_params)
    assert int(out["cold_batch"]) == C.sizeof(cold.cold_batch)
    assert int(out["cold_info"]) == C.sizeof(cold.cold_info)
    assert int(out["cold_config.max_ads_per_call"]) == cold.cold_config.max_ads_per_call.offset
    assert int(out["cold_config.flags"]) == cold.cold_config.flags.offset
    assert int(out["cold_config.chunk_ads"]) == cold.cold_config.chunk_ads.offset
    assert int(out["cold_batch.offs_host"]) == cold.cold_batch.offs_host.offset
    assert int(out["cold_info.device_bytes"]) == cold.cold_info.device_bytes.offset
    assert int(out["cold_group.cardinality"]) == cold.cold_group.cardinality.offset


def test_status_strings():
    L = _lib()
    for code in range(11):
        s = L.cold_status_string(code).decode()
        assert s and s != "unknown status"
    assert L.cold_status_string(99).decode() == "unknown status"


def test_host_validation_before_cuda():
    """Schema / shape errors are reported before any CUDA call (so they work without a GPU)."""
    import coldgen
    sch = coldgen.schema_tiny()
    with pytest.raises(cold.ColdError) as e:
        cold.Context(sch.groups, sch.k, (64, 3), precision="f32")
    assert e.value.name == "COLD_ERR_SHAPE"
    with pytest.raises(cold.ColdError) as e:
        cold.Context(sch.groups, 12, sch.widths, precision="f32")
    assert e.value.name == "COLD_ERR_UNSUPPORTED"
    bad = list(sch.groups)
    bad[6] = coldgen.Group("x", coldgen.CROSS, 10, None, 3, 0)      # refs swapped: AD as user_ref
    with pytest.raises(cold.ColdError) as e:
        cold.Context(bad, sch.k, sch.widths, precision="f32")
    assert e.value.name == "COLD_ERR_SHAPE"
    with pytest.raises(cold.ColdError) as e:
        cold.Context(sch.groups, sch.k, sch.widths, precision="f32", selected=[3, 1])
    assert e.value.name == "COLD_ERR_SHAPE"
    with pytest.raises(cold.ColdError) as e:
        cold.Context(sch.groups, sch.k, sch.widths, precision="f32", max_ads=0)
    assert e.value.name == "COLD_ERR_INVALID_ARG"


def test_no_cpu_fallback_without_gpu():
    """On a box without a GPU a valid configuration fails loudly (COLD_ERR_CUDA), never falls back."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import coldgen
    sch = coldgen.schema_tiny()
    with pytest.raises(cold.ColdError) as e:
        cold.Context(sch.groups, sch.k, sch.widths, precision="f32")
    assert e.value.name == "COLD_ERR_CUDA"


def test_sm100a_code_in_library():
    """The library carries sm_100a SASS with tcgen05 MMAs, TMA and TMEM loads."""
    _lib()
    sass = subprocess.run(["cuobjdump", "-sass", cold.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass and "UTMASTG" in sass
    elf = subprocess.run(["cuobjdump", "-lelf", cold.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in elf


def test_select_groups_host_helper():
    """cold_select_groups is host-only: top-K by mean SE weight, ties to the lower schema index,
    ascending output, checked against the oracle's definition."""
    import numpy as np

    import oracle
    _lib()
    rng = np.random.default_rng(3)
    for M in (1, 5, 32):
        s = np.round(rng.uniform(0, 1, M), 1)          # rounding forces ties
        for K in sorted({1, max(1, M // 2), M}):
            assert cold.select_groups(s, K) == oracle.select_groups(s, K)
    with pytest.raises(cold.ColdError):
        cold.select_groups(np.zeros(4), 5)

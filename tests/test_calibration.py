"""the B200 hardware profile measured by
tools/calibrate_profile.py loads through the reference's own simulator
(pipesim.get_profile / HardwareProfile.from_json, pipesim.py:33-105, 171-182)
and drives its schedules and savings report (pipesim.py:225-372). CPU only:
the reference is imported from baseline/_ref (the pip --target install) or,
in the build container, from /root/reference; skipped when neither exists."""

import glob
import json
import os
import sys

import pytest

from conftest import ROOT

PROFILE_KEYS = {"name", "t_pre_norm", "t_attn", "t_post_norm", "t_select", "t_expert_compute",
                "t_load_disk_per_expert", "t_load_mem_per_expert", "t_predict", "parallel_load_slots", "std"}


def _profiles():
    return sorted(glob.glob(os.path.join(ROOT, "profiles", "*_b200_hardware_profile.json")))


@pytest.fixture(scope="module")
def pipesim():
    for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(cand, "moepredict")):
            if cand not in sys.path:
                sys.path.insert(0, cand)
            import moepredict.pipesim as P
            return P
    pytest.skip("the reference package is not available here")


def test_profiles_have_the_reference_schema():
    paths = _profiles()
    assert paths, "no calibrated profile committed under profiles/"
    for p in paths:
        d = json.load(open(p))
        assert set(d) == PROFILE_KEYS, p
        assert d["t_attn"] > 0 and all(d[k] >= 0 for k in PROFILE_KEYS - {"name", "std", "parallel_load_slots"})
        assert d["parallel_load_slots"] >= 1


def test_profile_loads_and_drives_the_reference_simulator(pipesim):
    P = pipesim
    for path in _profiles():
        name = os.path.basename(path)[:-5]
        prof = P.get_profile(name, os.path.join(ROOT, "profiles"))
        assert prof == P.HardwareProfile.from_json(path)
        assert prof.t_predict > 0 and prof.full_load_ms(6, "memory") == 6 * prof.t_load_mem_per_expert
        # the prefetch window the B200 leaves for loading (pipesim.py:308-316)
        win = P.prefetch_window_ms(prof)
        assert win == pytest.approx(prof.t_attn + prof.t_post_norm + prof.t_select - prof.t_predict)
        assert P.stall_free(prof, 6, "memory") == (prof.full_load_ms(6, "memory") <= win)
        rep = P.savings_report(0.93, 0.85, [prof, P.get_profile("a100-80gb")], n_tokens=1000)
        assert rep["rows"][0]["profile"] == prof.name
        assert rep["rows"][0]["delta_ms_per_token"] > 0
        lat = {mode: P.schedule(prof, 6, mode, miss_count=2 if mode == "prefetch_miss" else 0).token_latency
               for mode in ("no_prefetch", "prefetch_hit", "prefetch_miss")}
        assert lat["prefetch_hit"] <= lat["prefetch_miss"] and lat["prefetch_hit"] <= lat["no_prefetch"]

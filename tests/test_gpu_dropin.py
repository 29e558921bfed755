"""The drop-in proof on the GPU: the UNMODIFIED reference's energy_expectation
(oracle/_ref, compiled from /root/reference) runs with the B200 backend
plugged into its ContractionBackend interface via include/qtng_backend.hpp
(serially, with jobs=4 worker threads, and under the reference's own
MixedBackend width dispatch) and reproduces its NaiveBackend energy."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_energy")


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/dropin_energy not built")
@pytest.mark.parametrize("n,seed,p", [(10, 7, 1), (12, 3, 2), (16, 1005, 2)])
def test_reference_driver_with_b200_backend(n, seed, p):
    out = subprocess.run([BIN, str(n), str(seed), str(p)], capture_output=True, text=True,
                         timeout=600, check=True).stdout
    r = json.loads(out.strip().splitlines()[-1])
    assert r["energy_b200"] == r["energy_naive"]
    assert r["energy_b200_jobs4"] == r["energy_naive"]
    assert r["energy_mixed"] == r["energy_naive"]
    assert r["records_b200"] == r["records_naive"] and r["all_records_b200"]
    assert r["mixed_bad_dispatch"] == 0 and r["mixed_gpu_records"] > 0
    assert r["peak_b200"] == r["peak_naive"]
    assert r["refusal"].startswith("edge (") and "exceeds cap 3" in r["refusal"]


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/dropin_energy not built")
def test_reference_driver_c2_timed(golden):
    """C2 through the per-bucket drop-in (7,857 qtng_contract_bucket round
    trips), serial and with 16 reference worker threads: the energy equals the
    reference's naive energy; the wall times are printed for the record."""
    c = golden["configs"]["C2"]
    out = subprocess.run([BIN, "time", "30", str(c["seed"]), "4", "16"], capture_output=True,
                         text=True, timeout=900, check=True).stdout
    r = json.loads(out.strip().splitlines()[-1])
    print("DROPIN", json.dumps(r))
    assert r["buckets"] == c["n_records"]
    assert r["energy_jobs1"] == c["energy_naive"]
    assert r["energy_jobsN"] == c["energy_naive"]

"""Model kernel traces (models.py) through the gpuos:: scheduler on the B200:
tensor-core conv/GEMM/GEMV bodies and STREAM bodies of ResNet-50 / BERT-base
/ Llama-3-8B decode.

* Mirror: the replay clock decides (the dispatch/completion log is the
  replay engine's, bit-exact with the reference's model) while every atom
  also executes on the GPU; every block ran exactly once on its TPC set.
* Live: configs #2 / #3 shapes complete every request with TPC placement
  inside each atom's set."""
from __future__ import annotations

import pytest

from paper_2504_15465_b200 import models, workloads

pytestmark = pytest.mark.gpu


def test_mirror_resnet50_and_bert_traces(api, cuda_device):
    cfg = {"name": "mirror-models", "device": {"gpc_count": 2, "tpcs_per_gpc": 37},
           "policy": "full_system", "horizon_ms": 30.0, "seed": 5,
           "scheduler": {"rightsizer": False, "dvfs": False, "stealing": True, "atomizer": True},
           "apps": [
               {"id": "rn50", "priority": "hp", "quota": 37, "slo_ms": 50.0,
                "arrival": {"times_ms": [0.0, 10.0]}, "kernels": models.resnet50_infer(1)},
               {"id": "bert", "priority": "be", "quota": 37,
                "arrival": {"times_ms": [0.0]}, "kernels": models.bert_base_infer(2)}]}
    r = api.run({"scenario": {"config": cfg}, "backend": "mirror", "log": True})
    v = r["verify"]
    assert v["ok"], v
    assert v["missing"] == v["duplicated"] == v["misplaced"] == 0
    # conv / GEMM / GEMV outputs sampled against float64 (verify_tensor)
    assert v["tensor_kernels"] > 0 and v["tensor_checked"] > 0 and v["tensor_bad"] == 0, v
    assert r["gpu_atoms"] == r["atoms"]["hp"] + r["atoms"]["be"] > 0
    replay = api.run({"scenario": {"config": cfg}, "backend": "replay", "log": True})
    assert r["log"] == replay["log"]


@pytest.mark.parametrize("name", ["infer4", "hybrid", "hybrid_real_attention"])
def test_live_model_configs_complete(api, cuda_device, name):
    cfg = (workloads.infer4(150.0) if name == "infer4"
           else workloads.hybrid(150.0, real_attention=name.endswith("attention")))
    req = {"scenario": {"config": cfg}, "backend": "b200", "device": "b200", "requests": True,
           "timeline": True, "verify": True, "b200": {"chunk_cap": 256, "trace": True},
           "set": {"block_revocation": True}}
    with api.Session(req) as s:
        s.run()
        r = s.run()
    v = r["verify"]
    assert v["ok"], v
    assert v["tensor_kernels"] > 0 and v["tensor_checked"] > 0, v
    for i, a in enumerate(r["report"]["apps"]):
        if a["high_priority"]:  # requests still in flight at the horizon are not counted
            assert a["completed"] > 0 and a["completed"] >= a["offered"] - 3
        else:  # a best-effort training iteration may outlast a 150 ms run: it ran blocks
            assert r["b200"]["work_us_per_app"][i] > 0
    tl = r["b200"]["timeline"]
    for m0, m1, t0, t1 in zip(tl["mask0"], tl["mask1"], tl["touched0"], tl["touched1"]):
        assert (t0 & ~m0) == 0 and (t1 & ~m1) == 0 and (t0 | t1) != 0


def test_live_decode_kernels_chain_on_the_device(api, cuda_device):
    """Llama-3-8B decode alone with chain_launches: nearly every kernel of a
    token is submitted before its predecessor's last block ends (it rides
    behind it on the device), only GEMVs start before their predecessor
    ends (early start behind a gate), and the token latency beats
    host-paced launches of the same trace on the same device."""
    import json
    import statistics

    cfg = workloads.without_apps(workloads.hybrid(200.0), "rn50_train")
    p50 = {}
    for chain in (False, True):
        req = {"scenario": {"config": cfg}, "backend": "b200", "device": "b200", "requests": True,
               "timeline": True, "b200": {"chunk_cap": 256},
               "set": {"block_revocation": True, "chain_launches": chain}}
        with api.Session(req) as s:
            s.run()
            r = s.run()
        lat = [json.loads(x)["latency_us"] for x in r["request_log"].splitlines() if json.loads(x)["completed"]]
        assert len(lat) >= 5
        p50[chain] = statistics.median(lat)
        if chain:
            tl = r["b200"]["timeline"]
            order = sorted(range(len(tl["kernel"])), key=lambda i: tl["kernel"][i])  # launch order
            pairs = [(a, b) for a, b in zip(order, order[1:])
                     if tl["dev_first"][b] - tl["dev_last"][a] < 100_000]  # same token
            early = sum(1 for a, b in pairs if tl["submit"][b] < tl["dev_last"][a])
            assert early >= 0.8 * len(pairs), (early, len(pairs))
            kern = models.llama3_8b_decode(1024)
            for a, b in pairs:  # only a GEMV starts early (behind its gate)
                if kern[tl["kernel"][b] % len(kern)]["body"]["kind"] != "gemv_bf16":
                    assert tl["dev_first"][b] >= tl["dev_last"][a]
    assert p50[True] < 0.9 * p50[False], p50

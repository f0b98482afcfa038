"""Regenerates the golden fixtures from the UNMODIFIED reference.

Run in the build container (needs /root/reference and `make -C oracle`):
    python tests/golden/make_golden.py

Writes, under tests/golden/:
  vectors.jsonl.gz            known answers of the pure policy functions
                              (oracle/_ref/ref_vectors)
  logs/<case>.log.gz          dispatch/completion logs ("D"/"C"/"A"/"E" lines,
                              oracle/harness/ref_golden.cpp) for short runs
  reports/<case>.json         run_scenario report + request log
  digests.json                sha256 of the full-length logs of every preset
                              x policy and of the feature ladder
  scenarios/*.json            scenario configs the cases use
Every case is (scenario args) -> output of the reference; tests replay the
same args through the B200 library's replay backend and compare bytes.
"""
from __future__ import annotations

import gzip
import hashlib
import json
import os
import random
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.path.join(ROOT, "oracle", "_ref")

# The smoke scenario of the reference's CLI tests (test_cli.cpp:16-31).
CLI_SMOKE = {
    "name": "cli-smoke", "device": {"gpc_count": 1, "tpcs_per_gpc": 4},
    "policy": "full_system", "horizon_ms": 50, "seed": 3, "scheduler": {"dvfs": False},
    "apps": [
        {"id": "hp", "priority": "hp", "quota": 2, "slo_ms": 20,
         "arrival": {"times_ms": [0, 10, 20, 30, 40]},
         "kernels": [{"blocks": 4, "block_us": 500, "s": 0.5, "occ": 1}]},
        {"id": "be", "priority": "be", "quota": 2, "arrival": "closed_loop",
         "kernels": [{"blocks": 8, "block_us": 1000, "s": 0.3, "occ": 2}]},
    ],
}


def random_scenario(seed: int) -> dict:
    """Seeded synthetic scenarios covering poisson / closed-loop / times_ms
    arrivals, synth_model and explicit kernels, right-sizing and DVFS."""
    rng = random.Random(seed)
    gpcs, per = rng.choice([(2, 4), (3, 6), (6, 9), (8, 9)])
    total = gpcs * per
    napps = rng.randint(2, 4)
    quotas = []
    left = total
    for i in range(napps):
        q = max(1, rng.randint(1, max(1, left // (napps - i))))
        quotas.append(q)
        left -= q
    apps = []
    for i in range(napps):
        hp = i == 0 or rng.random() < 0.3
        app = {"id": f"t{i}", "priority": "hp" if hp else "be", "quota": quotas[i]}
        if hp:
            app["slo_ms"] = rng.choice([5, 20, 60])
        kind = rng.random()
        if kind < 0.4:
            app["arrival"] = {"poisson_rps": rng.choice([20, 50, 200]), "seed_offset": rng.randint(0, 3)}
        elif kind < 0.7 and not hp:
            app["arrival"] = "closed_loop"
        else:
            app["arrival"] = {"times_ms": sorted(rng.uniform(0, 180) for _ in range(rng.randint(3, 12)))}
        if rng.random() < 0.5:
            app["workload"] = {"model": {
                "layers": rng.randint(1, 6),
                "blocks": {"uniform": [8, rng.choice([64, 512, 2000])]},
                "block_us": {"choice": [50, 200, 500, 1000]},
                "s": {"uniform": [0.0, 1.0]}, "occ": {"choice": [1, 2, 4]},
                "seed_offset": rng.randint(0, 5)}}
        else:
            app["kernels"] = [{"blocks": rng.randint(1, 1500), "block_us": rng.choice([20, 100, 500, 2000]),
                               "s": round(rng.random(), 2), "occ": rng.choice([1, 2, 4, 8])}
                              for _ in range(rng.randint(1, 4))]
        if not hp and rng.random() < 0.3:
            app["tpc_cap"] = rng.randint(1, total)
        apps.append(app)
    sched = {"stealing": rng.random() < 0.8, "atomizer": rng.random() < 0.8,
             "rightsizer": rng.random() < 0.5, "dvfs": rng.random() < 0.4,
             "atom_duration_us": rng.choice([250, 1000, 2000]),
             "steal_horizon_us": rng.choice([0, 0, 100, 500]),
             "max_outstanding_atoms": rng.choice([1, 2, 3])}
    return {"name": f"random-{seed}", "device": {"gpc_count": gpcs, "tpcs_per_gpc": per},
            "policy": "full_system", "horizon_ms": 200, "seed": seed, "scheduler": sched, "apps": apps}


# (case name, ref_golden args). Short horizons keep fixtures small.
def cases() -> list[tuple[str, list[str]]]:
    out = [("cli_smoke", ["--config", "scenarios/cli_smoke.json"])]
    for p in ("fig7", "inf-inf", "inf-train"):
        out.append((f"{p}_2s", ["--preset", p, "--horizon-ms", "2000"]))
    for pol in ("mps_like", "mig_like", "time_slice", "priority_only", "reef_like"):
        out.append((f"inf-inf_{pol}_1s", ["--preset", "inf-inf", "--policy", pol, "--horizon-ms", "1000"]))
    out.append(("fig7_sched_only_2s", ["--preset", "fig7", "--horizon-ms", "2000",
                                       "--set", "stealing=0", "--set", "atomizer=0"]))
    out.append(("fig7_steal_only_2s", ["--preset", "fig7", "--horizon-ms", "2000", "--set", "atomizer=0"]))
    out.append(("inf-train_rs_only_2s", ["--preset", "inf-train", "--horizon-ms", "2000",
                                         "--set", "stealing=0", "--set", "dvfs=0"]))
    for seed in range(1, 13):
        out.append((f"random_{seed}", ["--config", f"scenarios/random_{seed}.json"]))
    # The B200-form BASELINE configs the bench and the live runs use (short
    # horizons): #1 fig7-b200, #5 one 8-tenant set per rank, #2 infer4 and
    # #3 hybrid on random-init model kernel traces.
    for name in B200_SCENARIOS:
        out.append((name, ["--config", f"scenarios/{name}.json"]))
    return out


def b200_scenarios() -> dict[str, dict]:
    import sys

    sys.path.insert(0, ROOT)
    from paper_2504_15465_b200 import workloads

    return {"fig7_b200_x10": workloads.fig7_b200(10.0, 2000.0),
            "box8_rank0": workloads.tenant_set(0, 10.0, 500.0),
            "box8_rank1": workloads.tenant_set(1, 10.0, 500.0),
            "infer4_300ms": workloads.infer4(300.0),
            "hybrid_300ms": workloads.hybrid(300.0)}


B200_SCENARIOS = ("fig7_b200_x10", "box8_rank0", "box8_rank1", "infer4_300ms", "hybrid_300ms")


def digest_cases() -> list[tuple[str, list[str]]]:
    out = []
    for p in ("fig7", "inf-inf", "inf-train"):
        for pol in ("full_system", "mps_like", "mig_like", "time_slice", "priority_only", "reef_like"):
            out.append((f"{p}_{pol}", ["--preset", p, "--policy", pol]))
        for knobs in (["stealing=0", "atomizer=0"], ["atomizer=0"], ["rightsizer=1", "dvfs=1"]):
            args = ["--preset", p]
            for k in knobs:
                args += ["--set", k]
            out.append((f"{p}_{'_'.join(knobs)}", args))
    return out


def write_gz(path: str, data: bytes) -> None:
    with open(path, "wb") as raw, gzip.GzipFile(fileobj=raw, mode="wb", mtime=0) as f:
        f.write(data)


def ref(tool: str, args: list[str]) -> bytes:
    r = subprocess.run([os.path.join(REF, tool)] + args, cwd=HERE, capture_output=True, check=True)
    return r.stdout


def main() -> None:
    os.makedirs(os.path.join(HERE, "scenarios"), exist_ok=True)
    os.makedirs(os.path.join(HERE, "logs"), exist_ok=True)
    os.makedirs(os.path.join(HERE, "reports"), exist_ok=True)
    with open(os.path.join(HERE, "scenarios", "cli_smoke.json"), "w") as f:
        json.dump(CLI_SMOKE, f, indent=1)
    for seed in range(1, 13):
        with open(os.path.join(HERE, "scenarios", f"random_{seed}.json"), "w") as f:
            json.dump(random_scenario(seed), f, indent=1)
    for name, cfg in b200_scenarios().items():
        with open(os.path.join(HERE, "scenarios", f"{name}.json"), "w") as f:
            json.dump(cfg, f, separators=(",", ":"))
    write_gz(os.path.join(HERE, "vectors.jsonl.gz"), ref("ref_vectors", []))
    index = {}
    for name, args in cases():
        log = ref("ref_golden", args)
        write_gz(os.path.join(HERE, "logs", name + ".log.gz"), log)
        rep = ref("ref_golden", args + ["--report"])
        with open(os.path.join(HERE, "reports", name + ".txt"), "wb") as f:
            f.write(rep)
        index[name] = args
    digests = {}
    for name, args in digest_cases():
        digests[name] = {"args": args, "sha256": hashlib.sha256(ref("ref_golden", args)).hexdigest()}
    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump({"cases": index, "digests": digests}, f, indent=1, sort_keys=True)
    print(f"{len(index)} logged cases, {len(digests)} digests")


if __name__ == "__main__":
    main()

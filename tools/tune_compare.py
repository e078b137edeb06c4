"""Analytic vs device-timed tuning of one BASELINE program.

    python tools/tune_compare.py --prog scaled_0p125 --bind N=512,M=512,D=64 --outer 32,12,12

Runs the reference search (tilecc/tuner/tuner.py:143-206, analytic `score`) and
the same search with tuner.DeviceScorer (each candidate's sm_100a realisation
timed on this GPU), then re-times both picks with more repetitions and prints
one JSON line: the picks, their realisation keys, device microseconds, TFLOP/s
and the device pick's gain over the analytic pick.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prog", default="scaled_0p125")
    ap.add_argument("--bind", default="N=512,M=512,D=64")
    ap.add_argument("--outer", default="32,12,12")
    ap.add_argument("--budget", type=int, default=48)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--causal", action="store_true")
    a = ap.parse_args()

    from paper_2604_14825_b200.frontdoor import import_tilecc
    import_tilecc()
    from tilecc.autosched.scheduler import SchedulerOptions, run_autoscheduler
    from tilecc.ma.device import DEFAULT_DEVICE
    from tilecc.pipeline import frontend, probe_binding
    from tilecc.tuner import tuner as ref

    from paper_2604_14825_b200 import ma_ir, tuner
    from paper_2604_14825_b200.programs import PROGRAMS
    from paper_2604_14825_b200.recognize import recognize

    binding = {k: int(v) for k, v in (kv.split("=") for kv in a.bind.split(","))}
    outer = tuple(int(x) for x in a.outer.split(","))
    text = PROGRAMS[a.prog]
    bound, base = frontend(text, binding)
    _, probe = frontend(text, probe_binding(binding))
    seeds = [s.schedule for s in run_autoscheduler(base, DEFAULT_DEVICE, SchedulerOptions())]
    cfg = lambda: ref.TunerConfig(budget=a.budget, population=8, seed=a.seed)
    mk = "causal" if a.causal else "none"

    analytic = ref.search(seeds, base, probe, DEFAULT_DEVICE, cfg()).best()
    scorer = tuner.DeviceScorer(outer=outer, mask_kind=mk, reps=5)
    device = tuner.search(seeds, base, probe, DEFAULT_DEVICE, cfg(), scorer=scorer).best()

    final = tuner.DeviceScorer(outer=outer, mask_kind=mk, reps=21, warmup=3)
    out = {"prog": a.prog, "binding": binding, "outer": outer, "budget": a.budget,
           "device_realisations_timed": scorer.timed}
    for name, c in (("analytic_pick", analytic), ("device_pick", device)):
        us, _ = final(base, probe, seeds[c.seed_index], c.assignment, DEFAULT_DEVICE)
        mod = ma_ir.from_tilecc(tuner._lower(base, seeds[c.seed_index], c.assignment, DEFAULT_DEVICE))
        spec = recognize(mod)[0]
        flops = spec.flops(a.causal) * outer[0] * outer[1]
        out[name] = {"seed": c.seed_index, "assignment": c.assignment,
                     "realisation": list(tuner.realisation_key(spec, outer, mk)[8:]),
                     "device_us": us, "tflops": flops / (us * 1e-6) / 1e12}
    out["device_pick_speedup"] = out["analytic_pick"]["device_us"] / out["device_pick"]["device_us"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()

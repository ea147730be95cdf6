"""Print the Algorithm 4 / Algorithm 1 bench lines written by tools/alg4_ab.sh (tag as argv[1])."""
import json
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r2i"
for f in ("c2_alg4", "c2_alg1", "c4_alg4", "c4_alg1"):
    d = json.loads(open(f"gpurun_out/{tag}_bench_{f}.json").read().strip().splitlines()[-1])
    st = d["roofline"].get("stage_ms_per_step") or d.get("stage_ms_per_step")
    c = d["config"]
    print(f, round(d["value"]), round(d["ms_per_step"], 2), "e2e", round(d["e2e"]["value"]),
          {k: round(v, 2) for k, v in st.items()}, c.get("early_objects_per_query"),
          c.get("early_candidates_per_query"), c.get("recall"))

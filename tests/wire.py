"""Serialise a shard's host SoA back into the reference's /process wire JSON
(build_process_response schema, proj/src/handlers.cpp:57-91) — test helper."""
import json

ROLES = ["system", "user", "assistant", "tool"]


def to_responses(b, text="tool said \"hi\" \\ é"):
    starts = {}
    for k, t in enumerate(b.turns):
        starts.setdefault(int(t["traj"]), []).append(k)
    out = []
    for s in range(b.n_rollouts):
        traj = []
        for k in starts.get(s, []):
            t = b.turns[k]
            o, L, r = int(t["src_off"]), int(t["len"]), int(t["role"])
            ids = b.ids[o:o + L].tolist()
            traj.append({"input_ids": [] if r == 2 else ids, "logprobs": b.lp[o:o + L].tolist() if r == 2 else [],
                         "output_ids": ids if r == 2 else [], "role": ROLES[r], "text": text})
        out.append(json.dumps({"job_id": f"j{s}", "status": "DONE" if b.usable[s] else "FAILED",
                               "reward": float(b.reward[s]), "trajectory": traj,
                               "timings": {"init_seconds": 0.0}}).encode())
    return out

"""Request driver on top of the C ABI: prefill every request, then step + commit until done."""
from __future__ import annotations

from dataclasses import dataclass, field

from .focus import FocusContext


@dataclass
class GenLog:
    steps: int = 0
    decoded: int = 0
    per_step: list = field(default_factory=list)    # per step: list of commit dicts


def prefill_all(ctx: FocusContext, prompts, gen_len: int, rids=None):
    rids = list(range(len(prompts))) if rids is None else list(rids)
    for r in rids:
        ctx.focus_kv_append(r, prompts[r], gen_len)
    return rids


def generate(ctx: FocusContext, rids, max_steps: int = 1 << 30, keep_log: bool = True) -> GenLog:
    log = GenLog()
    live = list(rids)
    while live and log.steps < max_steps:
        ctx.focus_step_block(live)
        res = ctx.commit_results(live)
        log.steps += 1
        log.decoded += sum(r["n_new"] for r in res)
        if keep_log:
            log.per_step.append(res)
        live = [r["req_id"] for r in res if not r["finished"]]
    return log

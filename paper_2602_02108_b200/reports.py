"""Observability in the reference's formats.

* memory_report_to_json — paged_kv.cpp:13-22 (`nlohmann::json::dump()` of MemoryReport:
  keys in sorted order, no whitespace).
* dump_schedule_jsonl   — tiered_memory.cpp:28-45: a header line {"bandwidth_bytes_per_s": ...},
  then one object per ScheduleEvent with page / chunk / bytes omitted when negative / zero.
* emit_retrieval_csv    — chunktrain.cpp:115-130: one line `step,chunk,layer,global_query_page,page`
  per selected page, chunks in order, then layers, then query pages, pages in list order;
  global_query_page = chunk * pages_per_chunk + query page.
"""
from __future__ import annotations

import json


def memory_report_to_json(rep) -> str:
    d = {"device_bytes": int(rep.device_bytes), "host_bytes": int(rep.host_bytes), "grad_bytes": int(rep.grad_bytes),
         "pages": int(rep.pages), "reallocs": int(rep.reallocs), "copied_bytes": int(rep.copied_bytes)}
    return json.dumps(d, sort_keys=True, separators=(",", ":"))


def emit_retrieval_csv(out, step: int, chunks) -> None:
    """chunks: iterable of (chunk_index, per_layer) where per_layer[l] is a Selection or a list of
    per-query-page id lists (ChunkState::selected[layer], chunk_trainer.hpp:44)."""
    for index, per_layer in chunks:
        for layer, sel in enumerate(per_layer):
            lists = sel.lists() if hasattr(sel, "lists") else sel
            m = len(lists)
            for qp, ids in enumerate(lists):
                for page in ids:
                    out.write(f"{step},{index},{layer},{index * m + qp},{int(page)}\n")


def dump_schedule_jsonl(log, out) -> None:
    """tiered_memory.cpp:28-45 for a tiered_memory.ScheduleLog (nlohmann::json::dump: sorted keys, no
    whitespace, shortest round-trip doubles)."""
    out.write(json.dumps({"bandwidth_bytes_per_s": float(log.bandwidth_bytes_per_s)}, separators=(",", ":")) + "\n")
    for e in log.events:
        j = {"event": e.kind, "t": float(e.t), "layer": int(e.layer), "phase": e.phase}
        if e.page >= 0:
            j["page"] = int(e.page)
        if e.chunk >= 0:
            j["chunk"] = int(e.chunk)
        if e.bytes > 0:
            j["bytes"] = int(e.bytes)
        out.write(json.dumps(j, sort_keys=True, separators=(",", ":")) + "\n")

"""Observability in the reference's formats.

* memory_report_to_json — paged_kv.cpp:13-22 (`nlohmann::json::dump()` of MemoryReport:
  keys in sorted order, no whitespace).
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

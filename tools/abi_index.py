#!/usr/bin/env python3
"""Markdown index of every C-ABI export in include/flowreg_b200.h with the
reference interface it replaces: the file:line citations of the comment
directly above (or trailing) its prototype unless the curated entry below
says more;
"B200-specific" for exports with no reference counterpart.

    python tools/abi_index.py > /tmp/index.md
"""
import os
import re

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lines = open(os.path.join(root, "include", "flowreg_b200.h")).read().splitlines()
cite = re.compile(r"\b([A-Za-z_]+\.(?:py|md)):(\d+(?:-\d+)?(?:,\d+(?:-\d+)?)*)")
proto = re.compile(r"^\s*(?:int|int64_t|const char\*)\s+(frg_[a-z0-9_]+)\s*\(")

CURATED = {
    "frg_last_error": "B200-specific (error channel; the reference raises ValueError / RuntimeError)",
    "frg_version": "B200-specific",
    "frg_sample": "_kernels.py:222-251",
    "frg_dot": "fields.py:320-337",
    "frg_kkt_create": "kkt.py:139-162",
    "frg_kkt_set_interp_precision": "B200-specific (the north star's fp16 interpolation mode)",
    "frg_points_to_disp": "transport.py:37-45",
    "frg_tile_plan_count": "B200-specific (tile plans of the TMA engine; reference: per-point gathers, _kernels.py:191-219)",
    "frg_tile_plan": "B200-specific (tile plans of the TMA engine)",
    "frg_gather_planned": "interp.py:42-62 (with a prebuilt tile plan)",
    "frg_determinant": "fields.py:302-312",
    "frg_norm_inf": "fields.py:338-344",
    "frg_min_max_sum": "fields.py:320-344 (det F statistics, optimizer.py:276-279)",
    "frg_all_finite": "fields.py:160-205 (constructors' finiteness checks)",
    "frg_axpby": "fields.py:320-344 (vector algebra of optimizer.py:92-166)",
    "frg_kkt_destroy": "kkt.py:136 (context lifetime)",
    "frg_release_pool": "B200-specific (device buffer pool)",
    "frg_probe_arm": "B200-specific (bench measurement probe)",
    "frg_probe_read": "B200-specific (bench measurement probe)",
    "frg_peer_free": "PAPER.md:545 (peer windows, see frg_peer_alloc)",
    "frg_peer_open": "PAPER.md:545 (peer windows)",
    "frg_peer_close": "PAPER.md:545 (peer windows)",
    "frg_peer_register": "PAPER.md:545 (peer windows)",
    "frg_peer_unregister": "PAPER.md:545 (peer windows)",
    "frg_kkt_set_stream": "B200-specific (stream ordering)",
    "frg_kkt_set_images": "kkt.py:139-162",
    "frg_kkt_initial_mismatch": "kkt.py:139-162 (initial mismatch for the report, optimizer.py:197-281)",
    "frg_kkt_counters": "kkt.py:158-160",
    "frg_kkt_set_counters": "kkt.py:158-160",
    "frg_kkt_get": "kkt.py:166-187 (state fields the Python mirror exposes)",
    "frg_slab_departure": "transport.py:37-45 (one slab; PAPER.md:500-545)",
    "frg_slab_gather": "interp.py:42-62, transport.py:83-98 (one slab)",
    "frg_slab_adjoint_multiplier": "transport.py:105-135 (one slab)",
    "frg_slab_adjoint_step": "transport.py:105-135 (one slab)",
    "frg_slab_inc_first": "transport.py:147-176 (one slab)",
    "frg_slab_inc_step": "transport.py:147-176 (one slab)",
    "frg_slab_fd8_gradient": "diffops.py:98-106 (one slab)",
    "frg_slab_fd8_divergence": "diffops.py:117-129 (one slab)",
    "frg_slab_fft2": "diffops.py:44-73 (fftn, distributed: PAPER.md:507)",
    "frg_slab_fft1": "diffops.py:44-73 (fftn, distributed: PAPER.md:507)",
    "frg_slab_transpose": "diffops.py:44-73 (fftn, distributed: PAPER.md:507)",
    "frg_slab_spec_apply": "diffops.py:176-205,283-301 (split spectrum)",
    "frg_slab_spec_combine_mixed": "kkt.py:233-260, diffops.py:245-280 (alpha L a + P(b), split spectrum)",
    "frg_slab_spec_combine": "kkt.py:233-260, diffops.py:245-280 (alpha L a + P(b), split spectrum)",
    "frg_slab_grad_energy": "kkt.py:207-218",
    "frg_slab_body_force": "kkt.py:225-231 (one slab)",
    "frg_convert": "fields.py:77-80 (dtype conversion)",
    "frg_bind_plan": "B200-specific (tile plans of the slab path)",
    "frg_clear_plans": "B200-specific (tile plans of the slab path)",
}

section = "library"
rows = []
block, in_block = [], False
for i, ln in enumerate(lines):
    s = ln.strip()
    if not s:
        block = []
        continue
    if s.startswith("/* ----"):
        m = re.match(r"/\*\s*-+\s*(.*?)\s*-*\s*(\*/)?$", s)
        text = m.group(1).strip(" -") if m else ""
        section = text or None  # None: the block's first text line names it
        block = []
        in_block = not s.endswith("*/")
        continue
    if section is None and in_block:
        section = s.lstrip("* ").split(" (")[0]
    if s.startswith("/*") and not proto.match(ln):
        block = [s] if not in_block else block + [s]
        in_block = not s.endswith("*/")
        continue
    if in_block:
        block.append(s)
        in_block = not s.endswith("*/")
        continue
    pm = proto.match(ln)
    if pm:
        name = pm.group(1)
        tail, j = [], i
        while j < len(lines):
            tail.append(lines[j])
            if lines[j].rstrip().endswith((";", "*/")):
                break
            j += 1
        refs = sorted({f"{a}:{b}" for a, b in cite.findall(" ".join(block + tail))})
        rows.append((section, name, CURATED.get(name) or (", ".join(refs) if refs else "B200-specific")))
        block = []

print("| Section | Export | Reference interface replaced (file:line) |")
print("|---|---|---|")
for sec, name, refs in rows:
    print(f"| {sec} | `{name}` | {refs} |")

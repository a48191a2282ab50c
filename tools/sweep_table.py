"""Markdown table of a bench.py JSON line's per-format sweep (Mrays/s vs bytes/voxel)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().split("\n")[-1])
if len(sys.argv) > 2:  # bench.py --sweep --sweep-out FILE: the rows live in their own file
    d["sweep"] = json.load(open(sys.argv[2]))["rows"]
print(f"## {d['config']['workload']}\n")
print(f"headline: {d['config']['format']} {d['config']['variant']}: {d['value']} Mrays/s "
      f"({d['ms_per_step']} ms/frame, {d['config'].get('rays_per_frame', d['config'].get('rays'))} rays), e2e {d['e2e']['value']} Mrays/s; "
      f"clocks {d.get('clocks')}\n")
cb = d.get("cpu_baseline") or {}
if cb:
    print(f"oracle: {cb['value']:.3f} Mrays/s on {cb['cores']} host threads; parity sample {cb['parity_checked']} rays, "
          f"{cb['parity_mismatches']} mismatches\n")
print("| format | variant | kernel | Mrays/s | Mrays/s scheduled | B/voxel (device) | B/voxel (paper) | MiB | alg B/ray | sector B/ray | compulsory B/ray | DRAM B/ray (ncu) | HBM frac | cells/ray | descents/ray | SIMT bound | whole-level dedup gain | parity (mismatch/checked) |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for r in d.get("sweep", []):
    if "error" in r:
        print(f"| {r['format']} | — | error: {r['error']} |")
        continue
    print(f"| {r['format']} | {r['variant']} | {r.get('kernel', '—')} | {r['mrays_s']} | {r.get('mrays_s_scheduled') or '—'} | {r['bytes_per_voxel']} | {r['paper_bytes_per_voxel']} | "
          f"{r['mib']} | {r['alg_bytes_per_ray']} | {r.get('sector_bytes_per_ray', '—')} | "
          f"{r.get('compulsory_bytes_per_ray', '—')} | {r.get('dram_bytes_per_ray', '—')} | {r['roofline_frac']} | "
          f"{r['cells_per_ray']} | {r['descents_per_ray']} | {r['simt_bound']} | {r.get('wld_reduction') or '—'} | "
          f"{r.get('parity_mismatches', '—')}/{r.get('parity_checked', '—')} |")

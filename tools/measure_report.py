"""Write profiles/<tag>_measure.md from one tools/final_measure.sh run.

  python tools/measure_report.py gpurun_out/final r01

Inputs (all produced on the GPU box by tools/final_measure.sh): bench{1,2,4}.log,
bench_ref.log, measure_single.jsonl, measure_strong{1,2,4}.jsonl, timing{2,4}.log,
smi.txt, cpu.txt.  Also copies the raw files to profiles/<tag>_measure/.
"""
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def last_json(path):
    try:
        lines = [l for l in open(path).read().splitlines() if l.startswith("{")]
        return json.loads(lines[-1]) if lines else None
    except FileNotFoundError:
        return None


def jsonl(path):
    try:
        return [json.loads(l) for l in open(path) if l.startswith("{")]
    except FileNotFoundError:
        return []


def main():
    src, tag = sys.argv[1], sys.argv[2]
    out = []
    w = out.append
    w(f"# Measurements {tag} (B200, one tools/final_measure.sh run)\n")
    smi = open(os.path.join(src, "smi.txt")).read().strip() if os.path.exists(os.path.join(src, "smi.txt")) else ""
    cpu = open(os.path.join(src, "cpu.txt")).read().strip() if os.path.exists(os.path.join(src, "cpu.txt")) else ""
    w("All GPU numbers: CUDA events on the context stream after warm-up, max over ranks. "
      "GDOF/s counts local GLL points n_p = E(N+1)^3 (reading Q21). Raw files: "
      f"`profiles/{tag}_measure/`.\n")
    if smi:
        w("```\n" + smi + "\n" + cpu + "\n```\n")

    # ---- bench lines
    w("## bench.py (C2 per GPU, one PCG iteration per step, weak scaling)\n")
    w("| GPUs | value GDOF/s | ms/step | efficiency vs 1 GPU | Ax+gs GDOF/s (2-kernel) | Ax roofline frac | e2e GDOF/s | clocks MHz |")
    w("|---|---|---|---|---|---|---|---|")
    b1 = last_json(os.path.join(src, "bench1.log"))
    for P in (1, 2, 4):
        b = last_json(os.path.join(src, f"bench{P}.log"))
        if not b:
            continue
        eff = b["value"] / (P * b1["value"]) if b1 else float("nan")
        w(f"| {P} | {b['value']:.2f} | {b['ms_per_step']:.4f} | {eff:.3f} | "
          f"{b['ax_gs']['two_kernel']['gdofs']:.1f} | {b['roofline']['frac']:.3f} | "
          f"{b['e2e']['value']:.1f} | {b['clocks']['sm_mhz']:.0f} |")
    if b1:
        r = b1["roofline"]
        w("")
        w(f"Dominant kernel (1 GPU): `{r['kernel']}`, {r['bytes_per_pt']} B/pt algorithmic, "
          f"{r['avg_ms_per_apply'] * 1e3:.1f} us per application, achieved {r['achieved']:.0f} GB/s "
          f"= {r['frac']:.3f} of {r['peak']} GB/s ({r['peak_source']}); ncu DRAM traffic per launch "
          f"{r['traffic']}. Other kernels per step (ms): {json.dumps(r.get('other_kernels_ms_per_step'))}. "
          f"Ax only: {b1['ax_only']['gdofs']:.1f} GDOF/s. CPU oracle: {b1['cpu_baseline']['value']:.3f} "
          f"GDOF/s on {b1['cpu_baseline']['cores']} threads ({b1['cpu_baseline']['sample']}).\n")
    ref = last_json(os.path.join(src, "bench_ref.log"))
    if ref:
        w(f"`--impl reference` (the CPU oracle, the tier's reference arm): {ref.get('value')} {ref.get('unit')}, "
          f"{ref.get('cpu_baseline', {}).get('sample', '')}\n")

    # ---- single-GPU measurements
    rows = jsonl(os.path.join(src, "measure_single.jsonl"))
    byw = {r["what"]: r for r in rows if r.get("what") != "sweep"}
    if "triad" in byw:
        t = byw["triad"]
        w(f"## Denominators\n\nnominal 8000 GB/s; measured copy {t['copy_peak_GBps']} GB/s "
          f"(MEASURED_PEAKS.json); fp64 STREAM triad measured in this run: {t['GBps']:.0f} GB/s "
          f"(torch `add(b, c, alpha)`, 3 x 1 GiB vectors).\n")
    w("## Ax and Ax+gs on the BASELINE configs (1 GPU)\n")
    w("| config | n_p | Ax GDOF/s | Ax frac copy | Ax+gs GDOF/s (auto) | frac nominal | frac copy | frac triad | flat | chunks |")
    w("|---|---|---|---|---|---|---|---|---|---|")
    for key in ("C3_ops", "C4_ops_P1"):
        if key not in byw:
            continue
        d = byw[key]
        a, g = d["ax"], d["ax_gs"]
        w(f"| {key.split('_')[0]} | {d['n_p']} | {a['gdofs']} | {a['frac_copy']} | {g['gdofs']} | "
          f"{g['frac_nominal']} | {g['frac_copy']} | {g['frac_triad']} | "
          f"{d.get('ax_gs_flat', {}).get('gdofs')} | {d.get('ax_gs_chunks', {}).get('gdofs')} |")
    w("")
    if "C3_pcg_to_tol" in byw:
        d = byw["C3_pcg_to_tol"]
        w(f"**C3 PCG to tol {d['tol']}** (TGV pressure, 32^3 elements, N=7): {d['iters']} iterations, "
          f"{d['ms']} ms ({d['iter_per_s']} it/s, {d['gdofs']} GDOF/s), recursive residual "
          f"{d['res_final']:.3e}, true residual {d['res_true']:.3e}, e_inf vs p* after mean removal "
          f"{d['e_inf_vs_p*']:.2e}.\n")
    if "C4_pcg_P1" in byw:
        d = byw["C4_pcg_P1"]
        w(f"**C4 PCG, 1 GPU** (64^3 deformed, N=7, fixed {d['iters']} iterations): {d['iter_per_s']} it/s, "
          f"{d['gdofs']} GDOF/s.\n")
    sw = [r for r in rows if r.get("what") == "sweep"]
    if sw:
        w("## Polynomial-order sweep (1 GPU, n_p ~ 1.25e8 per GPU: E_axis = 500/(N+1))\n")
        w("| N | mesh | n_p | Ax GDOF/s | Ax frac copy | Ax+gs GDOF/s | Ax+gs B/pt | frac nominal | frac copy | setup s |")
        w("|---|---|---|---|---|---|---|---|---|---|")
        for d in sw:
            w(f"| {d['N']} | {'x'.join(map(str, d['mesh']))} | {d['n_p']} | {d['ax']['gdofs']} | "
              f"{d['ax']['frac_copy']} | {d['ax_gs']['gdofs']} | {d['ax_gs_B_per_pt']} | "
              f"{d['ax_gs']['frac_nominal']} | {d['ax_gs']['frac_copy']} | {d['setup_s']} |")
        w("")

    # ---- strong scaling
    st = {}
    for P in (1, 2, 4):
        for r in jsonl(os.path.join(src, f"measure_strong{P}.jsonl")):
            st[(r["what"], P)] = r
    if st:
        w("## Strong scaling (C3 and C4 split into z-slabs over P GPUs, NVLink peer memory)\n")
        w("| config | P | Ax+gs GDOF/s | PCG it/s | PCG GDOF/s | PCG efficiency T1/(P TP) |")
        w("|---|---|---|---|---|---|")
        for cfg in ("C3_strong", "C4_strong"):
            base = st.get((cfg, 1))
            for P in (1, 2, 4):
                d = st.get((cfg, P))
                if not d:
                    continue
                eff = d["pcg_gdofs"] / (P * base["pcg_gdofs"]) if base else float("nan")
                w(f"| {cfg.split('_')[0]} | {P} | {d['ax_gs_gdofs']} | {d['pcg_iter_per_s']} | "
                  f"{d['pcg_gdofs']} | {eff:.3f} |")
        w("")
    for P in (2, 4):
        t = next((r for r in jsonl(os.path.join(src, f"timing{P}.log")) if "P" in r), None)
        if t:
            keys = [k for k in t if k.startswith("p2p_noov") or k.startswith("nccl_ov") or k == "ax_only_us"]
            w(f"Per-phase times at P={P} (C2 per GPU, us; `p2p_noov` = default NVLink path, "
              f"`nccl_ov` = NCCL with Alg. 1 overlap): " + ", ".join(f"{k} {t[k]}" for k in keys) + "\n")

    dst = os.path.join(ROOT, "profiles", f"{tag}_measure")
    os.makedirs(dst, exist_ok=True)
    for f in os.listdir(src):
        if f.endswith((".log", ".jsonl", ".txt")):
            shutil.copy(os.path.join(src, f), os.path.join(dst, f))
    path = os.path.join(ROOT, "profiles", f"{tag}_measure.md")
    with open(path, "w") as f:
        f.write("\n".join(out) + "\n")
    print(path)


if __name__ == "__main__":
    main()

"""Per-kernel HBM evidence (ncu --set full) for the non-pole kernels of a step:
    python tools/summarize_aux.py gpurun_out/<rep>.ncu-rep <D> > profiles/<name>.md
Algorithmic bytes per launch (DESIGN.md 6.2/6.3) vs dram bytes, achieved GB/s vs the measured
HBM copy bandwidth in MEASURED_PEAKS.json."""
import csv
import io
import json
import os
import subprocess
import sys

rep, D = sys.argv[1], int(sys.argv[2])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
n = D * D
algo = {  # bytes that must move per launch (3 fields)
    "fft_rows_fwd_kernel": 3 * n * (8 + 8),         # real rows in, half-spectrum rows out
    "fft_cols_fwd_kernel": 3 * n * (8 + 8),         # half spectrum in, rows l <= D/2 out (apply path)
    "fft_cols_inv_kernel": 3 * n * (8 + 8),         # Hermitian accumulator: half columns in, half out
    "fft_rows_fwd16_kernel": 3 * n * (8 + 8),
    "fft_cols_fwd16_kernel": 3 * n * (8 + 8),       # apply path: rows l <= D/2 of the spectrum only
    "fft_cols_inv16_kernel": 3 * n * (8 + 8),
    "fft_cols_cl_kernel": 3 * n * (8 + 8),          # cluster column passes (forward: half out)
    "fft_rows_inv16_kernel": 3 * n * (8 + 8),
    "fft_rows_inv_kernel": 3 * n * (8 + 8),         # half-spectrum rows in, real rows out
    "finish_kernel": None,   # chunk partials in (chunks x 32 B per pair) + 48 B per k <= D/2 mode out
    "fixup_k0_kernel": None,
}
def col(name):
    return h.index(name) if name in h else None
ik, it = col("Kernel Name"), col("gpu__time_duration.sum")
ir, iw = col("dram__bytes_read.sum"), col("dram__bytes_write.sum")
unit_r = rows[1][ir]
print(f"# Non-pole kernels at {D}^2 (ncu --set full, cold cache)\n")
print(f"HBM peak: {peak} GB/s (MEASURED_PEAKS.json `hbm_gbs`, of measured).\n")
print("| kernel | time (us) | DRAM read+write (MB) | algorithmic (MB) | DRAM GB/s | DRAM of measured peak | algorithmic GB/s | algorithmic of measured peak |")
print("|---|---|---|---|---|---|---|---|")
scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
for r in rows[2:]:
    name = r[ik].split("(")[0].replace("void ", "").replace("rexi::", "")
    base = name.split("<")[0].strip()
    t_us = float(r[it].replace(",", ""))  # usecond in --page raw (ncu default unit)
    u = rows[1][it]
    t_us = t_us / 1e3 if u == "nsecond" else (t_us * 1e3 if u == "msecond" else t_us)
    mb = float(r[ir].replace(",", "")) * scale.get(rows[1][ir], 1e-6) + \
        float(r[iw].replace(",", "")) * scale.get(rows[1][iw], 1e-6)
    al = algo.get(base)
    gbs = mb * 1e6 / (t_us * 1e-6) / 1e9
    alg = (al / 1e6) / t_us * 1e6 / 1e3 if al else float('nan')   # algorithmic GB/s
    print(f"| `{name}` | {t_us:.1f} | {mb:.2f} | {al / 1e6 if al else float('nan'):.2f} | {gbs:.0f} | {gbs / peak:.2f} | {alg:.0f} | {alg / peak:.2f} |")

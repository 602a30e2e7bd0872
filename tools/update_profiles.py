"""Copy the round-end captures of tools/gpu_final1.sh (gpurun_out/final/; or
`python tools/update_profiles.py <gpurun_out subdir> <file prefix>`) into profiles/:
ncu summaries of the dominant kernels, the launch lists, and profiles/ncu_summary.json
(the per-launch DRAM traffic bench.py reports as roofline.traffic)."""
import json, shutil, subprocess, sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "gpurun_out" / (sys.argv[1] if len(sys.argv) > 1 else "final")
PREFIX = sys.argv[2] if len(sys.argv) > 2 else "r1_final"
PROF = ROOT / "profiles"
CASES = [("mix_rand_psgd_float32_L64_d25557032", "c2_rad", 12),
         ("mix_d1d_float32_L64_d25557032", "c4_d1d", 12),
         ("mix_rand_psgd_bfloat16_L64_d25557032", "c2_rad_bf16", 6)]
L, D = 64, 25_557_032


def num(s):
    v, u = s.split()
    return float(v) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1.0,
                       "us": 1e-3}[u]


def main():
    out = {}
    for key, name, bpp in CASES:
        rep = SRC / f"prof_{name}.ncu-rep"
        js = PROF / f"{PREFIX}_{name}_ncu.json"
        txt = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(rep)],
                             capture_output=True, text=True, check=True).stdout
        js.write_text(txt)
        d = json.loads(txt)
        r, w = num(d["dram__bytes_read.sum"]), num(d["dram__bytes_write.sum"])
        alg = bpp * L * D
        out[key] = {"kernel": d["kernel"],
                    "source": f"profiles/{js.name} (ncu --set full, 1 launch, round-end capture)",
                    "dram_bytes_read": r, "dram_bytes_write": w, "dram_bytes_per_launch": r + w,
                    "algorithmic_bytes_per_launch": alg,
                    "traffic_over_algorithmic": round((r + w) / alg, 4),
                    "duration_ms_ncu": num(d["gpu__time_duration.sum"])}
    (PROF / "ncu_summary.json").write_text(json.dumps(out, indent=1) + "\n")
    for f in ("launches_default.csv", "launches_normals_c2.csv"):
        shutil.copy(SRC / f, PROF / f"{PREFIX}_{f}")
    print(json.dumps({k: v["traffic_over_algorithmic"] for k, v in out.items()}))


if __name__ == "__main__":
    main()

"""profiles/<tag>_summary.md (+ bench line, launch list, traffic json, pytest log) from a tools/gpu_round_evidence.sh run.

usage: python tools/round_summary.py TAG"""
import json
import shutil
import subprocess
import sys

tag = sys.argv[1]
for f in (f"{tag}_bench_c4.json", f"{tag}_launches_c4.csv", f"{tag}_pytest.log"):
    shutil.copy(f"gpurun_out/{f}", f"profiles/{f}")
subprocess.run([sys.executable, "tools/traffic_json.py", f"profiles/{tag}_launches_c4.csv", "4", "100000000",
                f"profiles/{tag}_traffic_c4.json"], check=True, stdout=subprocess.DEVNULL)
d = json.loads(open(f"profiles/{tag}_bench_c4.json").read().strip().splitlines()[-1])
tab = subprocess.run([sys.executable, "tools/launches.py", f"profiles/{tag}_launches_c4.csv"], capture_output=True,
                     text=True).stdout
e, r = d["e2e"], d["roofline"]
npass = open(f"profiles/{tag}_pytest.log").read().strip().splitlines()[-1]
tr = f"{r['traffic'] / 1e9:.2f} GB per launch ({r['traffic_source']})" if r.get("traffic") else "none committed"
out = f"""# Profile {tag}: config 4 (10^8 float64 keys, int32 payload)

GPU: {open(f'gpurun_out/{tag}_gpu.txt').read().strip().splitlines()[-1]}

`python bench.py --steps 20 --warmup 5` (CUDA events, warm, L2 flushed between steps, clocks {d['clocks']['sm_mhz']:.0f}/{d['clocks']['sm_max_mhz']:.0f} MHz, throttle reasons {d['clocks']['reasons']}):
**{d['ms_per_step']:.3f} ms per sort = {d['value'] / 1e9:.2f} G keys/s**; whole sort {d['sort_roofline']['achieved_gbs']:.0f} GB/s of algorithmic traffic (64 B/key) = {100 * d['sort_roofline']['frac']:.1f} % of the measured {r['peak']} GB/s.
Dominant kernel `{r['kernel']}`: {r['launches_per_step']:.0f} launches per sort over {r['records_per_step']:.3g} records, {r['alg_bytes_per_launch'] / 1e9:.2f} GB algorithmic per launch in {r['launch_ms']:.3f} ms = {r['achieved']:.0f} GB/s = **{100 * r['frac']:.1f} % of peak per launch** ({100 * r['one_pass_frac']:.1f} % when only one pass over n is credited); ncu DRAM traffic {tr}.
Phases (ms per sort): {json.dumps(d['phases_ms_per_step'])}; stats {d['stats']}; {d['gpu_launches']} launches per sort.

End to end (host buffers, copies inside the timed region): `SortPipeline` stream of sorts **{e['ms_per_step']:.2f} ms per step = {e['value'] / 1e9:.2f} G keys/s** ({e['vs_pipeline_floor']:.2f}x the max(H2D, D2H) = {e['pipeline_floor_ms']:.1f} ms floor; H2D {e['h2d_gbs']:.1f} GB/s, D2H {e['d2h_gbs']:.1f} GB/s measured alone); one `zsort` of host data in series {e['single_sort']['ms_per_step']:.1f} ms ({e['single_sort']['vs_copy_floor']:.2f}x its H2D + D2H floor of {e['single_sort']['copy_floor_ms']:.1f} ms).
Paper mapping (exact Eq. 1 at level 1): {d['paper_mapping']['ms_per_step']:.2f} ms; config 5 at 2^31 keys on this GPU: {d['c5_single_gpu']['ms_per_step']:.1f} ms ({d['c5_single_gpu']['keys_per_s'] / 1e9:.1f} G keys/s, {100 * d['c5_single_gpu']['sort_roofline']['frac']:.1f} % of the 80 B/key roofline, {d['c5_single_gpu']['structural_check_violations']} violations); torch.sort(stable)+gather {d['comparators']['torch.sort(stable=True)+gather']['ms_per_step']:.2f} ms ({d['comparators']['torch.sort(stable=True)+gather']['ours_speedup']:.2f}x slower).
CPU baseline (oracle port, 1 core): {d['cpu_baseline']['value'] / 1e6:.1f} M keys/s.

GPU tests at this build: `profiles/{tag}_pytest.log` ({npass}).

Launch list: `ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none python tools/prof_sort.py --config 4` (one profiled sort after a warm-up sort; cold-cache, serialised: compare shares).

```
{tab}```

`ncu --set full` of the same sort (same kernels for this config): `profiles/r02ba_ncu_key_c4.txt` (per-launch metrics and stall ratios), `profiles/r02ba_ncu_lines_scatter_c4.txt`, `profiles/r02ba_ncu_lines_finish_c4.txt` (instructions and stall samples per source line), `profiles/r02ba_ncu_smem_scatter_c4.txt` (shared-memory wavefronts per source line); read in DESIGN.md 4.3.
"""
open(f"profiles/{tag}_summary.md", "w").write(out)
print(out[:900])

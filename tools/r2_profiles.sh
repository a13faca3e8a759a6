#!/bin/bash
# Copy the evidence of a tools/r2_final.sh + tools/ncu_programs.sh run (TAG) from
# gpurun_out/ into profiles/r02_* (profiling aid).   tools/r2_profiles.sh r02e
TAG=$1
tail -1 gpurun_out/${TAG}_pytest_gpu.txt
cp gpurun_out/${TAG}_pytest_gpu.txt profiles/r02_pytest_gpu.txt
tail -1 gpurun_out/${TAG}_bench_c3.json > profiles/r02_bench_c3.json
cp gpurun_out/${TAG}_all_configs.jsonl profiles/r02_all_configs.jsonl
CMD="PT_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-online"
python tools/ncu_summary.py list gpurun_out/${TAG}_launches_c3.csv "$CMD" > profiles/r02_launches_c3.json
for k in A M AM; do
  python tools/ncu_summary.py rep gpurun_out/${TAG}_ncu_c3_${k}.ncu-rep "c3 ${k} executor program alone (ncu --set full, launch 3 of 4)" "ncu --set full --import-source on --clock-control none -k regex:pt_exec_kernel -s 2 -c 1 python tools/ncu_target.py c3 $k 4" > /tmp/ncu_c3_${k}.json
  python tools/ncu_summary.py rep gpurun_out/${TAG}t_ncu_c2_${k}.ncu-rep "c2 ${k} executor program alone, tile-major dense kernels (ncu --set full, launch 3 of 4)" "ncu --set full --import-source on --clock-control none -k regex:pt_exec_kernel -s 2 -c 1 python tools/ncu_target.py c2 $k 4" > /tmp/ncu_c2t_${k}.json
done
python - "$TAG" <<'PY'
import json,subprocess,csv,io,sys
TAG=sys.argv[1]
def extra(path):
    out=subprocess.run(["ncu","-i",path,"--page","raw","--csv","--print-units","base"],capture_output=True,text=True).stdout
    rows=list(csv.reader(io.StringIO(out))); h=rows[0]; v=rows[2]
    return {n:v[i]+" "+rows[1][i] for i,n in enumerate(h) if n in ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed","dram__bytes.sum.per_second")}
PEAK=6552.0
for tag,pre,rep,note in (("r02_ncu_c3_programs","/tmp/ncu_c3_",f"gpurun_out/{TAG}_ncu_c3_","round-2 executor, final"),
                     ("r02_ncu_c2_programs_tiles","/tmp/ncu_c2t_",f"gpurun_out/{TAG}t_ncu_c2_","round-2 dense path, final: dense kernels stored tile-major and streamed by the 16-row Y tasks")):
    res={"note":note,"peak_hbm_gbs_measured":PEAK,"programs":{}}
    for k in ("A","M","AM"):
        d=json.load(open(f"{pre}{k}.json")); l=d["launches"][0]
        l.update(extra(f"{rep}{k}.ncu-rep"))
        t=float(l["gpu__time_duration.sum"].split()[0])
        l["dram_gbs"]=round(l["traffic_bytes"]/t,1); l["dram_frac_of_measured_peak"]=round(l["traffic_bytes"]/t/PEAK,3)
        res["programs"][k]={"command":d["command"],**l}
        print(tag,k,l["gpu__time_duration.sum"],l["traffic_bytes"],l["dram_gbs"],l["dram_frac_of_measured_peak"])
    json.dump(res,open(f"profiles/{tag}.json","w"),indent=1)
t=json.load(open("profiles/ncu_traffic.json")); t["c3"]=json.load(open("profiles/r02_ncu_c3_programs.json"))["programs"]["AM"]["traffic_bytes"]; t["c2"]=json.load(open("profiles/r02_ncu_c2_programs_tiles.json"))["programs"]["AM"]["traffic_bytes"]; json.dump(t,open("profiles/ncu_traffic.json","w"),indent=1)
for l in open("profiles/r02_all_configs.jsonl"):
    d=json.loads(l); name=d["config"]["workload"].split(":")[0]
    print(name, round(d["value"],3), d["parity"]["iterations"], d["parity"]["trace_rel_err_vs_reference"], round(d["roofline"]["frac"],3), round(d["solve"]["solve_frac"],3))
d=json.loads(open("profiles/r02_bench_c3.json").read()); print("c3 bench", d["value"], d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["achieved"], d["roofline"]["launch_ms_avg"], d["cpu_baseline"]["value"], d.get("online_pipeline",{}).get("device_total_ms"), d["clocks"])
k=json.load(open("profiles/r02_launches_c3.json"))["kernels"]; print({n.split("(")[0][-20:]:v["share"] for n,v in k.items()})
PY

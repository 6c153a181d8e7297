cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for d in desk paper; do
timeout 300 python tools/stream_check.py --dims $d --steps 80 > gpurun_out/r2j_stream_$d.json 2> gpurun_out/r2j_stream_$d.err
LTFB_NO_STREAM=2 timeout 300 python tools/stream_check.py --dims $d --steps 80 > gpurun_out/r2j_launch_$d.json 2> gpurun_out/r2j_launch_$d.err
timeout 300 python tools/stream_check.py --dims $d --steps 8 --n 8000 --time-steps 1000 > gpurun_out/r2j_stime_$d.json 2> gpurun_out/r2j_stime_$d.err
LTFB_NO_STREAM=1 timeout 300 python tools/stream_check.py --dims $d --steps 8 --n 8000 --time-steps 1000 > gpurun_out/r2j_ltime_$d.json 2> gpurun_out/r2j_ltime_$d.err
python - <<PY
import json
d="$d"
a=json.load(open(f'gpurun_out/r2j_stream_{d}.json')); b=json.load(open(f'gpurun_out/r2j_launch_{d}.json'))
print(d, "stream", a["stream"], b["stream"], "ctas", a["wide_ctas"], b["wide_ctas"], "identical:", a["records"]==b["records"], a["fwd_hash"]==b["fwd_hash"], a["disc_hash"]==b["disc_hash"], a["inv_hash"]==b["inv_hash"], a["eval"]==b["eval"])
print(d, "ms/step stream", json.load(open(f"gpurun_out/r2j_stime_{d}.json")).get("ms_per_step"), "launched", json.load(open(f"gpurun_out/r2j_ltime_{d}.json")).get("ms_per_step"))
PY
done

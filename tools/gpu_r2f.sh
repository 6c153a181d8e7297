cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/stream_check.py --steps 80 > gpurun_out/r2f_stream.json 2> gpurun_out/r2f_stream.err
LTFB_NO_STREAM=2 timeout 300 python tools/stream_check.py --steps 80 > gpurun_out/r2f_launch.json 2> gpurun_out/r2f_launch.err
LTFB_STREAM_PROF=1 timeout 120 python tools/stream_check.py --steps 8 --n 8000 --time-steps 200 > gpurun_out/r2f_prof.json 2> gpurun_out/r2f_prof.err
timeout 300 python tools/stream_check.py --steps 8 --n 8000 --time-steps 1000 > gpurun_out/r2f_stream_time.json 2> gpurun_out/r2f_stream_time.err
python - <<'PY'
import json
a=json.load(open('gpurun_out/r2f_stream.json')); b=json.load(open('gpurun_out/r2f_launch.json'))
print("stream", a["stream"], b["stream"], "ctas", a["wide_ctas"], b["wide_ctas"])
print("records identical:", a["records"]==b["records"], "hashes", a["fwd_hash"]==b["fwd_hash"], a["disc_hash"]==b["disc_hash"], a["inv_hash"]==b["inv_hash"], "eval", a["eval"]==b["eval"])
d=json.load(open("gpurun_out/r2f_stream_time.json")); print("stream ms/step", d.get("ms_per_step"))
PY
tail -n 2 gpurun_out/r2f_prof.err; tail -n 3 gpurun_out/r2f_stream.err

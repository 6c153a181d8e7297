cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/stream_check.py --steps 80 > gpurun_out/r2c_stream.json 2> gpurun_out/r2c_stream.err; echo "rc=$?" >> gpurun_out/r2c_stream.err
LTFB_NO_STREAM=2 timeout 300 python tools/stream_check.py --steps 80 > gpurun_out/r2c_launch.json 2> gpurun_out/r2c_launch.err; echo "rc=$?" >> gpurun_out/r2c_launch.err
timeout 300 python tools/stream_check.py --steps 8 --n 8000 --time-steps 1000 > gpurun_out/r2c_stream_time.json 2> gpurun_out/r2c_stream_time.err
LTFB_NO_STREAM=1 timeout 300 python tools/stream_check.py --steps 8 --n 8000 --time-steps 1000 > gpurun_out/r2c_launch_time.json 2> gpurun_out/r2c_launch_time.err
python - <<'PY'
import json
a=json.load(open('gpurun_out/r2c_stream.json')); b=json.load(open('gpurun_out/r2c_launch.json'))
print("stream", a["stream"], b["stream"], "ctas", a["wide_ctas"], b["wide_ctas"])
print("records identical:", a["records"]==b["records"], "hashes", a["fwd_hash"]==b["fwd_hash"], a["disc_hash"]==b["disc_hash"], a["inv_hash"]==b["inv_hash"], "eval", a["eval"]==b["eval"])
for x,y in zip(a["records"], b["records"]):
    if x!=y: print("first diff", x, y); break
for f in ("r2c_stream_time.json","r2c_launch_time.json"):
    try: d=json.load(open("gpurun_out/"+f)); print(f, d.get("stream"), d.get("ms_per_step"))
    except Exception as e: print(f, "failed", e)
PY
for f in gpurun_out/r2c_*.err; do echo "== $f"; tail -n 4 $f; done

cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
LTFB_STREAM_DEBUG=1 timeout 120 python tools/stream_check.py --steps 32 > gpurun_out/r2d_stream.json 2> gpurun_out/r2d_stream.err; echo "rc=$?" >> gpurun_out/r2d_stream.err
LTFB_NO_STREAM=2 timeout 120 python tools/stream_check.py --steps 32 > gpurun_out/r2d_launch.json 2> gpurun_out/r2d_launch.err
python - <<'PY'
import json
a=json.load(open('gpurun_out/r2d_stream.json')); b=json.load(open('gpurun_out/r2d_launch.json'))
print("wall", a["wall_s"], b["wall_s"])
for x,y in list(zip(a["records"], b["records"]))[:20]:
    print(x==y, x[3:6], y[3:6])
PY
cat gpurun_out/r2d_stream.err | tail -n 20

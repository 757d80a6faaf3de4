# quick GPU iteration: parity tests + kernel-only bench numbers
# usage: bash tools/gpu_quick.sh [pytest -k expr]
set -o pipefail
if [ -n "$1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$1" 2>&1 | tail -4
else
  timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
fi
timeout 300 python bench.py --no-e2e --no-cpu --no-plugin --steps 20 > gpurun_out/quick.json 2> gpurun_out/quick.err || tail -20 gpurun_out/quick.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/quick.json"))
print("value", round(d["value"], 1), "ms", round(d["ms_per_step"], 4),
      "decode_ms", round(d["decode"]["ms"], 4), "encode_kernel_ms", round(d["encode"]["kernel_ms"], 4),
      "model_ms", round(d["model_build"]["ms"], 4),
      "sb14 eager", round(d["sb14"]["ms_per_step_eager"], 4), "sb14 dec", round(d["sb14"]["decode_ms"], 4),
      "sb14 enc", round(d["sb14"]["encode_kernel_ms"], 4))
PY

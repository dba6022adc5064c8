# one compute-sanitizer tool per call: bash scripts/gpu_san.sh memcheck|synccheck|initcheck|racecheck
T=$1
mkdir -p gpurun_out
python -c "from paper_1609_01479_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 600 python scripts/sanitize_cases.py > gpurun_out/san_plain_$T.log 2>&1 && \
timeout 2400 compute-sanitizer --tool $T --print-limit 50 python scripts/sanitize_cases.py > gpurun_out/san_$T.log 2>&1
echo san=$?; tail -25 gpurun_out/san_$T.log

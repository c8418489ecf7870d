for a in "--no-cpu-baseline" "" "--no-cpu-baseline"; do
PRGPU_TIMING_LOG=1 timeout 900 python bench.py --steps 10 --warmup 3 $a > gpurun_out/bv.log 2>&1
echo "args=[$a] $(grep -c . gpurun_out/bv.log) lines"; grep "offsets h2d" gpurun_out/bv.log | tail -6 | awk '{print $5}' | tr '\n' ' '; echo; grep "e2e split" gpurun_out/bv.log | tr '\n' ' ' | cut -c1-400; echo
python -c "import json;d=json.loads(open('gpurun_out/bv.log').read().strip().splitlines()[-1]);print('e2e ms', d['e2e']['ms_per_step'])"
done

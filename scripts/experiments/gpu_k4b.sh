mkdir -p gpurun_out
run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 6 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
bq() { timeout 300 python bench.py --config $1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'GTEPS', round(d['ms_per_step'],3), 'ms/step')"; }
for v in 0 1; do echo "c5 k4cfg=$v $(PRGPU_K4CFG=$v run c5)"; done
for a in 0 1; do for b in 0 1; do for c in 0 1; do echo "c2 K8=$a K4=$b K2=$c $(PRGPU_K8CFG=$a PRGPU_K4CFG=$b PRGPU_K2CFG=$c bq c2)"; done; done; done
for b in 0 1; do for c in 0 1; do echo "c5 K4=$b K2=$c $(PRGPU_K4CFG=$b PRGPU_K2CFG=$c bq c5)"; done; done
P="python scripts/prof_pull.py --config c5 --launches 3"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:pull_kernel<.int.2, .int.2," -s 2 -c 2 -o gpurun_out/c5_pull2 $P > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
tail -2 gpurun_out/ncu_c5.log

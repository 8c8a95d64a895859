#!/usr/bin/env bash
# One GPU-box pass (run under gpurun from the repo root):
#   GPU parity tests, smoke(), the bench line (both arms), the ncu launch
#   list of the bench command and one `ncu --set full` capture of K2.
# Everything lands in gpurun_out/; summaries worth keeping go to profiles/.
#   STAGES="tests smoke bench ref launches full" (default: all)
set -u
mkdir -p gpurun_out
STAGES=${STAGES:-"tests smoke bench ref launches full"}
NCU=${NCU:-ncu}
has() { case " $STAGES " in *" $1 "*) return 0;; esac; return 1; }

nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/nproc.txt

if has tests; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest -m gpu exit $?" | tee -a gpurun_out/status.txt
fi
if has smoke; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
  echo "smoke exit $?" | tee -a gpurun_out/status.txt
fi
if has bench; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench exit $?" | tee -a gpurun_out/status.txt
fi
if has ref; then
  timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
  echo "bench ref exit $?" | tee -a gpurun_out/status.txt
fi
if has launches; then
  timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/launches_bench.log 2>&1
  echo "ncu launches exit $?" | tee -a gpurun_out/status.txt
fi
if has full; then
  timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:k2_soa -s 3 -c 1 \
      -f -o gpurun_out/prof_k2 \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_k2.log 2>&1
  echo "ncu full exit $?" | tee -a gpurun_out/status.txt
fi

#!/usr/bin/env bash
# ncu --set full captures (source-level) of the top kernels, run under
# gpurun from the repo root. Reports + CSV source pages land in gpurun_out/.
#   KERNELS="k2 hinsert aos" (default: k2)
set -u
mkdir -p gpurun_out
KERNELS=${KERNELS:-k2}
TAG=${TAG:-r2}
has() { case " $KERNELS " in *" $1 "*) return 0;; esac; return 1; }
cap() { # name, kernel regex, bench args...
  local name=$1 re=$2; shift 2
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$re" -s 3 -c 1 \
      -f -o gpurun_out/${name}_${TAG} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" \
      > gpurun_out/${name}_${TAG}.log 2>&1
  echo "$name ncu exit $?"
  ncu -i gpurun_out/${name}_${TAG}.ncu-rep --page source --csv --print-source=cuda,sass \
      > gpurun_out/${name}_${TAG}_source.csv 2>/dev/null
  ncu -i gpurun_out/${name}_${TAG}.ncu-rep --page raw --csv > gpurun_out/${name}_${TAG}_raw.csv 2>/dev/null
  ncu -i gpurun_out/${name}_${TAG}.ncu-rep --page details > gpurun_out/${name}_${TAG}_details.txt 2>/dev/null
}
has k2 && cap k2 k2_soa
has hinsert && cap hinsert h_insert --hosts
has aos && cap aos k2_gen --input aos
if has hpost; then
  # the per-host median passes (h_coarse, h_fine) of one step
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:h_coarse|h_fine|h_collect" -s 9 -c 3 \
      -f -o gpurun_out/hpost_${TAG} python bench.py --hosts --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
      --no-pageable --no-adapter --no-extras > gpurun_out/hpost_${TAG}.log 2>&1
  echo "hpost ncu exit $?"
  ncu -i gpurun_out/hpost_${TAG}.ncu-rep --page source --csv --print-source=cuda,sass \
      > gpurun_out/hpost_${TAG}_source.csv 2>/dev/null
  ncu -i gpurun_out/hpost_${TAG}.ncu-rep --page details > gpurun_out/hpost_${TAG}_details.txt 2>/dev/null
fi

if has small; then
  # one capture each of the step's small kernels (K1 plan, finalize)
  timeout 1200 ncu --set full --clock-control none --import-source on \
      -k "regex:k2b_fine|k3a_median|k3b_final|k_sample|k_hot_select|k_table_slots" -s 18 -c 6 \
      -f -o gpurun_out/small_${TAG} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
      > gpurun_out/small_${TAG}.log 2>&1
  echo "small ncu exit $?"
  ncu -i gpurun_out/small_${TAG}.ncu-rep --page details > gpurun_out/small_${TAG}_details.txt 2>/dev/null
fi
if has launches; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_${TAG}.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/launches_${TAG}.log 2>&1
  echo "launches exit $?"
fi
if has hlaunches; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/hlaunches_${TAG}.csv \
      python bench.py --hosts --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-pageable --no-adapter \
      > gpurun_out/hlaunches_${TAG}.log 2>&1
  echo "hlaunches exit $?"
fi
if has hbench; then
  python bench.py --hosts --no-cpu-baseline --no-pageable --no-adapter > gpurun_out/hbench_${TAG}.json 2>&1
  echo "hbench exit $?"
fi
exit 0

#!/usr/bin/env bash
# Builds the SPECSIM_ADAMW_VARIANT probe libraries here (no GPU needed):
#   scripts/adamw_probe.sh build
# and runs them on the GPU box:  scripts/adamw_probe.sh run
# Variants: 0 production (256-bit accesses); on the 128-bit epilogue: 1 no p/m/v
#           loads, 2 only the bf16 store, 3 plain (no streaming hint) loads / stores,
#           4 all 8 row groups hoisted, 5 as shipped before the 256-bit epilogue;
#           6: production epilogue with the state folded into an L2-resident
#           1 Mi-element window (same SM <-> L2 traffic, no HBM state stream);
#           7 / 8: production epilogue + L2 prefetch of the state (whole
#           half-tile row before the accumulator wait / one chunk ahead)
cd "$(dirname "$0")/.."
if [ "$1" = build ]; then
  mkdir -p probe
  for v in ${VARIANTS:-1 2 3 4 5 6 7 8}; do
    extra=-DSPECSIM_ADAMW_VARIANT=$v
    [ $v = 6 ] && extra="-DSPECSIM_ADAMW_WINDOW=1048576"
    [ $v = 7 ] && extra="-DSPECSIM_ADAMW_PREFETCH=1"
    [ $v = 8 ] && extra="-DSPECSIM_ADAMW_PREFETCH=2"
    make -C paper_2602_05145_b200/csrc -j8 OUT=$PWD/probe/libv$v.so BUILD=build_v$v \
      EXTRA="$extra" > /dev/null || exit 1
  done
  exit 0
fi
mkdir -p gpurun_out
for v in ${VARIANTS:-0 1 2 3 4 5 6}; do
  lib=$PWD/probe/libv$v.so; [ $v = 0 ] && lib=$PWD/paper_2602_05145_b200/libspecsim_draft.so
  TAG=v$v SPECSIM_LIB=$lib timeout 300 python scripts/adamw_probe.py
done | tee gpurun_out/adamw_probe.jsonl

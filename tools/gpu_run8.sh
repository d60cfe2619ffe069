# knob sweep on config 5 (COUNT_HASH, D2): housekeeping period, donation spacing, low-water mark
run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --no-secondary --no-e2e --steps 5 > gpurun_out/bench8_$tag.log 2>&1; }
run base X=1
run ps64 TPGEN_LIB_VARIANT=ps64
run sm128 TPGEN_SPLIT_MIN=128
run sm512 TPGEN_SPLIT_MIN=512
run lw4k TPGEN_LOW_WATER=4096
run lw64k TPGEN_LOW_WATER=65536
run base2 X=1

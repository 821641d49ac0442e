#!/bin/bash
# One documented gpurun driver script (replaces the round-1 one-off cmd*.sh files).
#
#   gpurun --timeout 3000 -- 'bash tools/gpu_round.sh TAG [STEPS...]'
#
# TAG names the outputs (gpurun_out/TAG_*).  STEPS (default: build tests smoke bench) pick
# what runs, in order:
#   build    compile libtps.so for sm_100a on the box
#   tests    pytest -m gpu (full GPU parity suite)
#   quick    pytest -m gpu on the fast files only (pipeline, fused update, ABI step-wise)
#   smoke    __graft_entry__.smoke()
#   bench    bench.py default line (C5, S=1) + the reference arm
#   configs  tools/bench_configs.py (per-config one-GPU numbers incl. C2/C4 V vs I)
#   launches ncu launch list of one bench epoch window + its summary
#   gemm     tools/gemm_bench.py microbenchmarks at the bench shape (clock / power sampled)
#   ncu      ncu --set full of one launch each of the fwd / dgrad / blend / fused-update GEMMs
#   sanitize compute-sanitizer racecheck/synccheck/memcheck on small pipeline runs
#   resnet   ResNet GPU tests, C4 one-GPU numbers with the BN ReLU bit mask + specialised col2im
#            on and off (A/B), and the ResNet-50 per-kernel launch list with DRAM bytes
#   vgg      VGG-16 (C3, S = 1) per-kernel launch list with DRAM bytes (mid-run window)
#   fdab     parity suites with the forward / input-gradient split-K on (TPS_SPLITK_FD=1) and
#            C1-C3 one-GPU numbers with it on and off
#   vggab    conv / VGG parity tests, C3 one-GPU numbers with the tile-starved weight gradients
#            unfused (default) and fused (TPS_FUSE_ALL=1)
# Every step runs under its own timeout so one hang cannot eat the box.
set -u
TAG=${1:?tag}; shift
STEPS=${*:-build tests smoke bench}
mkdir -p gpurun_out
O=gpurun_out/${TAG}
for s in $STEPS; do
  case $s in
    build)
      python -c "import __graft_entry__ as g; g.build()" > ${O}_build.log 2>&1 ;;
    tests)
      timeout 2700 python -m pytest tests -q -m gpu --timeout=1500 -p no:cacheprovider --durations=12 > ${O}_tests.log 2>&1 ;;
    quick)
      timeout 1500 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_fused_update.py tests/test_gpu_stepwise.py -q -m gpu --timeout=900 -p no:cacheprovider > ${O}_quick.log 2>&1 ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1 ;;
    bench)
      timeout 900 python bench.py 2>${O}_bench.err | tail -1 > ${O}_bench.json
      timeout 900 python bench.py --impl reference --steps 2 --warmup 3 2>/dev/null | tail -1 > ${O}_ref.json ;;
    configs)
      timeout 1500 python tools/bench_configs.py --graph --out ${O}_configs.json > ${O}_configs.log 2>&1 ;;
    launches)
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 2500 -c 600 --csv \
        --log-file ${O}_launches.csv python bench.py --steps 1 --warmup 1 --epoch-mb 16 --no-cpu-baseline --no-e2e --no-v > /dev/null 2>&1
      python tools/launches_summary.py ${O}_launches.csv ${O}_launches_summary.json "bench.py C5 S=1, one epoch window" > /dev/null 2>&1 ;;
    gemm)
      timeout 600 python tools/gemm_bench.py --modes 0,1,2,3,4,7,8,9 --seconds 1.0 > ${O}_gemm.txt 2>&1 ;;
    ncu)
      # one launch each of fwd / dgrad / blended dgrad / fused wgrad + update at the C5 shapes
      # (summarised on the box with stall reasons; only the dominant kernel's report is kept, so
      # gpurun_out stays under the 64 MiB copy-back limit)
      for m in 0 1 3 4; do
        timeout 400 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 \
          -o ${O}_mode$m python tools/gemm_bench.py --modes $m --iters 1 > ${O}_ncu_mode$m.log 2>&1
        python tools/ncu_summary.py ${O}_mode$m.ncu-rep --stalls --json ${O}_ncu_mode$m.json > /dev/null 2>&1
        [ $m = 4 ] || rm -f ${O}_mode$m.ncu-rep
      done ;;
    sanitize)
      for tool in racecheck synccheck memcheck; do
        TPS_SANITIZE=1 timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 \
          python -m pytest tests/test_gpu_sanitize.py -q -m gpu -p no:cacheprovider > ${O}_san_${tool}.log 2>&1
        echo "exit $?" >> ${O}_san_${tool}.log
      done ;;
    resnet)
      timeout 1500 python -m pytest tests/test_gpu_resnet_ops.py tests/test_gpu_resnet.py tests/test_gpu_resnet50_ops.py \
        -q -m gpu --timeout=900 -p no:cacheprovider > ${O}_resnet_tests.log 2>&1
      for rep in 1 2; do
        timeout 600 python tools/bench_configs.py --graph --only C4 --out ${O}_c4_new$rep.json > ${O}_c4_new$rep.log 2>&1
        TPS_RELU_MASK=0 TPS_COL2IM_GENERIC=1 timeout 600 python tools/bench_configs.py --graph --only C4 \
          --out ${O}_c4_old$rep.json > ${O}_c4_old$rep.log 2>&1
      done
      timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
        --csv --log-file ${O}_r50_launches.csv python tools/profile_resnet.py --mb 1 > ${O}_r50_prof.log 2>&1
      python tools/ncu_launch_bw.py ${O}_r50_launches.csv --json ${O}_r50_launches_bw.json > ${O}_r50_bw.txt 2>&1 ;;
    vgg)
      timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
        -s 1500 -c 450 --csv --log-file ${O}_vgg_launches.csv python tools/bench_configs.py --only "C3 VGG-16 CIFAR S=1" \
        > ${O}_vgg_prof.log 2>&1
      python tools/ncu_launch_bw.py ${O}_vgg_launches.csv --json ${O}_vgg_launches_bw.json > ${O}_vgg_bw.txt 2>&1 ;;
    vggab)
      timeout 1200 python -m pytest tests/test_gpu_conv.py tests/test_gpu_resnet_ops.py \
        "tests/test_gpu_fullsize.py::test_c3_vgg16_four_stage" -q -m gpu --timeout=900 -p no:cacheprovider \
        > ${O}_vgg_tests.log 2>&1
      for rep in 1 2; do
        timeout 600 python tools/bench_configs.py --graph --only C3 --out ${O}_c3_new$rep.json > ${O}_c3_new$rep.log 2>&1
        TPS_FUSE_ALL=1 timeout 600 python tools/bench_configs.py --graph --only C3 --out ${O}_c3_old$rep.json \
          > ${O}_c3_old$rep.log 2>&1
      done ;;
    fdab)
      TPS_SPLITK_FD=1 timeout 1500 python -m pytest tests/test_gpu_conv.py tests/test_gpu_pipeline.py \
        tests/test_gpu_fused_update.py tests/test_gpu_stepwise.py tests/test_gpu_ipc.py tests/test_gpu_graph.py \
        "tests/test_gpu_fullsize.py::test_c3_vgg16_four_stage" -q -m gpu --timeout=900 -p no:cacheprovider \
        > ${O}_fd_tests.log 2>&1
      for c in C2 C3; do
        TPS_SPLITK_FD=1 timeout 900 python tools/bench_configs.py --graph --only $c --out ${O}_fd_on_$c.json \
          > ${O}_fd_on_$c.log 2>&1
        timeout 900 python tools/bench_configs.py --graph --only $c --out ${O}_fd_off_$c.json > ${O}_fd_off_$c.log 2>&1
      done ;;
    *) echo "unknown step $s" ;;
  esac
done

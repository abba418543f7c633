# A/B of the exact comparator (K4): parity tests with the variant, then throughput at config-3 and config-4 shapes
for v in "$@"; do
  RIANN_LIB=$PWD/_ab/lib_$v.so timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "exact_tc or exact_field or coherency" > gpurun_out/k4_${v}_pytest.log 2>&1; echo "$v pytest rc=$?"; tail -1 gpurun_out/k4_${v}_pytest.log
done
for rep in 1 2; do for v in "$@"; do
  echo "$v cfg3"; RIANN_LIB=$PWD/_ab/lib_$v.so timeout 600 python tools/bench_exact.py --cfg 3 --m 262144 --simt-m 256 2>&1 | tail -1 | cut -c1-400
  echo "$v cfg4"; RIANN_LIB=$PWD/_ab/lib_$v.so timeout 600 python tools/bench_exact.py --cfg 4 --m 524288 --simt-m 256 2>&1 | tail -1 | cut -c1-400
done; done

# Round-end evidence on one GPU: GPU tests, the bench line (no ncu in it),
# the reference arm, and the ncu launch list of the same bench command.
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1; echo rc=$? >> gpurun_out/final_pytest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo rc=$? >> gpurun_out/final_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo rc=$? >> gpurun_out/final_ref.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-comparator --no-configs --no-ncu > gpurun_out/final_ncu.log 2>&1; echo ncu_rc=$? >> gpurun_out/final_ncu.log
python tools/parity_campaign.py gpurun_out/final_parity_campaign.json > gpurun_out/final_parity_campaign.log 2>&1; echo rc=$? >> gpurun_out/final_parity_campaign.log

SEL='not full and not full_size and not graph'
for f in test_gpu_fwd test_gpu_bwd test_gpu_int8_out test_gpu_train; do
timeout 900 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 100000 \
  python -m pytest tests/$f.py -q -x -k "$SEL" -p no:cacheprovider > gpurun_out/rc_$f.log 2>&1; echo rc=$? >> gpurun_out/rc_$f.log
grep -E "Race reported|Write Thread|Read Thread|RACECHECK SUMMARY| at .* in " gpurun_out/rc_$f.log | sed 's/Thread ([0-9,]*)//; s/+0x[0-9a-f]*//; s/block ([0-9,]*)//; s/0x[0-9a-f]*//g' | sort | uniq -c | sort -rn > gpurun_out/rc_${f}_uniq.txt
done

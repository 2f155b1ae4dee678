cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1
for t in "tests/test_gpu_tileset.py" "tests/test_gpu_layers.py" "tests/test_gpu_verify.py -k 'not corrupted'" "tests/test_gpu_persistent.py -k 'not case4 and not reference'" "tests/test_gpu_umma.py -k 'tc and (mkn2 or mkn3 or mkn5 or mkn8)'" "tests/test_gpu_pair.py -k tc" "tests/test_gpu_glue_layers.py" "tests/test_gpu_sharded.py -k 'gcn and 2708'"; do
  echo "== memcheck $t" >> gpurun_out/r2_sanitizers.txt
  eval timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest $t -x -q -p no:cacheprovider 2>&1 | grep -E "ERROR SUMMARY|passed|failed|Error" | tail -3 >> gpurun_out/r2_sanitizers.txt
done
echo "== racecheck fbb_tc" >> gpurun_out/r2_sanitizers.txt
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_umma.py -x -q -k "tc and mkn3 and 32" -p no:cacheprovider 2>&1 | grep -E "RACECHECK SUMMARY|ERROR SUMMARY|passed|failed|hazard" | tail -3 >> gpurun_out/r2_sanitizers.txt
echo "== synccheck fbb_tc" >> gpurun_out/r2_sanitizers.txt
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_umma.py -x -q -k "tc and mkn3 and 32" -p no:cacheprovider 2>&1 | grep -E "ERROR SUMMARY|passed|failed" | tail -3 >> gpurun_out/r2_sanitizers.txt
cat gpurun_out/r2_sanitizers.txt

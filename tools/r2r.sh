# full-size Reddit parity (opt-in test) + compute-sanitizer memcheck / racecheck on the small parity cases
mkdir -p gpurun_out/r2r
( time TANGO_FULL_REDDIT=1 timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -k reddit > gpurun_out/r2r/reddit_parity.log 2>&1 ) 2>> gpurun_out/r2r/reddit_parity.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_layer.py -q -x -k "c0b_h2 or ragged or hd512" > gpurun_out/r2r/memcheck.log 2>&1; echo rc=$? >> gpurun_out/r2r/memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_layer.py -q -x -k "ragged and not recompute" > gpurun_out/r2r/racecheck.log 2>&1; echo rc=$? >> gpurun_out/r2r/racecheck.log
timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_layer.py -q -x -k "ragged and not recompute" > gpurun_out/r2r/synccheck.log 2>&1; echo rc=$? >> gpurun_out/r2r/synccheck.log

timeout 600 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_frontend.py tests/test_gpu_int8_out.py -q -x 2>&1 | tail -1
for lib in new old; do
 if [ $lib = old ]; then export QFB_LIB_PATH=$PWD/ab/libqfb_old.so; else unset QFB_LIB_PATH; fi
 echo -n "$lib c5 f32 "; python tools/c5_probe.py 8 f32
 echo -n "$lib c5 f16 "; python tools/c5_probe.py 8 f16
 echo -n "$lib 1f f32 "; python tools/c5_probe.py 1 f32
 echo -n "$lib 1f f16 "; python tools/c5_probe.py 1 f16
done
unset QFB_LIB_PATH

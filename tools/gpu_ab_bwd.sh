for r in 1 2; do for lib in new old; do
 if [ $lib = old ]; then export QFB_LIB_PATH=$PWD/ab/libqfb_old.so; else unset QFB_LIB_PATH; fi
 for d in f32 f16; do echo -n "$lib "; python tools/bwd_only_probe.py $d; done
done; done

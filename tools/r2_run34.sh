mkdir -p gpurun_out
timeout 1500 python tools/wsplit_ab.py --config c3wn --fracs 0.25,0.3,0.4 --reps 2 --no-uwalk 2>/dev/null
timeout 600 python tools/wsplit_ab.py --config c2 --fracs 0.25,0.4 --no-uwalk 2>/dev/null

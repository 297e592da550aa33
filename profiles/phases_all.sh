# per-phase device times of the BASELINE configs (FSR and SSR)
timeout 300 python profiles/phases.py moving 400 250 40000
timeout 300 python profiles/phases.py static 400 250 20000
timeout 300 python profiles/phases.py sensor 1000 1000 20000
timeout 300 python profiles/phases.py range 400 250 1000000 fsr

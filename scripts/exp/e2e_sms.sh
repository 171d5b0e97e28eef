# Does the kernel's SM footprint slow the DMA in the pinned e2e pipeline?
for cap in 0 74 37 148 0; do echo -n "GAES_SMS_CAP=$cap "; GAES_SMS_CAP=$cap python scripts/exp/e2e_ab.py; done

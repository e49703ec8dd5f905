"""B200-native WeatherMesh-3 forecast hot path (drop-in for the reference `gridcast` forecast API).

Host layer in Python mirrors gridcast's encode / process / decode / rollout / forecast API; the compute
runs in libwm3.so (hand-written sm_100a kernels behind the C ABI of include/wm3.h).
"""

__version__ = "0.1.0"

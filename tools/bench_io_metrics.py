"""Measure the SURVEY 8f widenings at full scale: LMTW load straight to the device (3.06 GB of float64
parameters), host LMTW load for comparison, and the device verification metrics over all 157 decoded planes of
a 0.25 deg forecast (per-plane RMSE + blur in one launch each, evaluation.plane_scores)."""
import os, sys, tempfile, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_22235_b200.model as M
from paper_2503_22235_b200 import evaluation as EV
from paper_2503_22235_b200.serialization import load_params_device, load_params_file, save_params_file

cfg = M.full_scale_config()
params = M.init_model_params(cfg, seed=0, zero_residual=False)
host = {k: v.values for k, v in params.items()}
nbytes = sum(v.nbytes for v in host.values())
d = tempfile.mkdtemp(dir="/tmp")
path = os.path.join(d, "full.lmtw")
t0 = time.perf_counter()
save_params_file(path, host)
t_save = time.perf_counter() - t0
os.system("sync")
t0 = time.perf_counter()
dev = load_params_device(path)
torch.cuda.synchronize()
t_dev = time.perf_counter() - t0
t0 = time.perf_counter()
hp = load_params_file(path)
t_host = time.perf_counter() - t0
ok = all(torch.equal(dev[k].cpu(), torch.from_numpy(hp[k]).float()) for k in list(hp)[:20])
print(f"LMTW {len(host)} tensors, {nbytes / 1e9:.2f} GB: save {t_save:.2f} s; load_params_device {t_dev:.2f} s "
      f"({nbytes / t_dev / 1e9:.1f} GB/s); load_params_file (host) {t_host:.2f} s; spot-check equal: {ok}")
del dev, hp
g = cfg.grid
rng = np.random.default_rng(1)
st = M.WeatherState(0, torch.from_numpy(rng.standard_normal((cfg.surface_in, g.rows, g.cols)).astype(np.float32)).cuda(),
                    torch.from_numpy(rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)).astype(np.float32)).cuda())
dec = M.decode(M.encode(st, params, cfg), params, cfg)
pred = torch.cat([dec.surface.device, dec.atmos.device.reshape(-1, g.rows, g.cols)])
truth = pred + 0.1 * torch.randn_like(pred)
EV.plane_scores(pred, truth, g, 2000.0)
torch.cuda.synchronize()
t0 = time.perf_counter()
rmse, blur = EV.plane_scores(pred, truth, g, 2000.0)
torch.cuda.synchronize()
t_eval = time.perf_counter() - t0
print(f"device verification: {pred.shape[0]} planes of {g.rows}x{g.cols}: RMSE + blur in {t_eval * 1e3:.1f} ms "
      f"(median rmse {np.median(rmse):.4f})")
os.remove(path)

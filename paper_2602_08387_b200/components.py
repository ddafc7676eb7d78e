"""Registered components of the training step (the drop-in boundary).

Interfaces follow the paper's object-graph model through
the reference's registry-factory contract:

  interface   variant          builds
  ---------   -------------    -----------------------------------------------
  dataset     packed_memmap    packed.PackedReader over an existing CFPKD001 file
  dataset     synthetic        a seeded synthetic CFPKD001 file (markov / uniform)
  sampler     sequential       data.Sampler(shuffle=False)
  sampler     permuted         data.Sampler(shuffle=True, seed)  (make_permutation)
  dataloader  packed_gpu       data.PackedDataLoader (resident or staged feed)
  model       gpt2 | llama     model.DecoderLM from a preset or explicit shape
                               (precision "bf16" training / "fp32" parity mode)
  optimizer   adamw_fused      optim.AdamWConfig (fused sharded AdamW on the GPU)
  trainer     fsdp_spmd        trainer.SPMDTrainer (the "gym")
  planner     fsdp_comm        comm_planner plan for a model shape (unit sizing)
  planner     fsdp_comm_calibrated   the same with (alpha, B) fitted to a measured NVLink sweep
  tokenizer   byte | whitespace | bpe   tokenizers.load_tokenizer (C++ encoder)
  pipeline    tokenize         a configured run_pipeline job (C++ thread pool)

``default_registry()`` returns a registry with all of them; a user adds a new
model architecture with ``register_component``.
"""

from __future__ import annotations

import os

from .config_graph import FactoryDescriptor, ParamSpec, Registry

P = ParamSpec


def _dataset_packed(path):
    from .packed import open_packed

    return open_packed(path)


def _dataset_synthetic(path, n_tokens, vocab_size, kind="markov", seed=0, doc_len=1024):
    from .data import make_synthetic_packed
    from .packed import open_packed

    if not os.path.exists(path):
        tmp = f"{path}.tmp{os.getpid()}"
        make_synthetic_packed(tmp, n_tokens, vocab_size, doc_len=doc_len, kind=kind, seed=seed)
        os.replace(tmp, path)
    return open_packed(path)


def _sampler_seq():
    from .data import Sampler

    return Sampler(shuffle=False)


def _sampler_perm(seed=0):
    from .data import Sampler

    if seed < 0:
        raise ValueError("seed must be a uint64 (>= 0)")
    return Sampler(shuffle=True, seed=seed)


def _dataloader(dataset, batch_size, seq_len, sampler=None, feed="resident"):
    from .data import PackedDataLoader

    return PackedDataLoader(dataset, batch_size, seq_len, sampler, feed)


def _model(arch):
    def build(preset=None, n_layer=None, d_model=None, n_head=None, n_kv_head=None, d_ff=None, vocab_size=None,
              max_seq_len=None, tie_embeddings=None, norm_eps=None, rope_theta=None, init_std=None,
              precision="bf16", activation_checkpointing=False):
        from dataclasses import replace

        from .model import PRESETS, DecoderLM, ModelConfig

        explicit = dict(n_layer=n_layer, d_model=d_model, n_head=n_head, n_kv_head=n_kv_head, d_ff=d_ff,
                        vocab_size=vocab_size, max_seq_len=max_seq_len, tie_embeddings=tie_embeddings,
                        norm_eps=norm_eps, rope_theta=rope_theta, init_std=init_std)
        explicit = {k: v for k, v in explicit.items() if v is not None}
        if preset is not None:
            cfg = PRESETS[preset]
            if cfg.arch != arch:
                raise ValueError(f"preset {preset!r} is a {cfg.arch} model, not {arch}")
            cfg = replace(cfg, **explicit)
        else:
            if arch == "gpt2":
                explicit.setdefault("n_kv_head", explicit.get("n_head"))
            cfg = ModelConfig(arch=arch, **explicit)
        return DecoderLM(cfg, precision, activation_checkpointing)

    return build


_MODEL_PARAMS = (P("preset", "string", required=False), P("n_layer", "int", required=False),
                 P("d_model", "int", required=False), P("n_head", "int", required=False),
                 P("n_kv_head", "int", required=False), P("d_ff", "int", required=False),
                 P("vocab_size", "int", required=False), P("max_seq_len", "int", required=False),
                 P("tie_embeddings", "bool", required=False), P("norm_eps", "float", required=False),
                 P("rope_theta", "float", required=False), P("init_std", "float", required=False),
                 P("precision", "string", required=False, default="bf16"),
                 P("activation_checkpointing", "bool", required=False, default=False))


def _optimizer(lr=3e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1, grad_clip=1.0, warmup_steps=10):
    from .optim import AdamWConfig

    return AdamWConfig(lr, beta1, beta2, eps, weight_decay, grad_clip, warmup_steps)


def _trainer(model, optimizer, dataloader, steps=20, seed=0, blocks_per_unit=1, init_device="cpu",
             log_every=0, metrics_path=None):
    from .trainer import SPMDTrainer

    return SPMDTrainer(model, optimizer, dataloader, steps=steps, seed=seed, blocks_per_unit=blocks_per_unit,
                       init_device=init_device, log_every=log_every, metrics_path=metrics_path)


def _planner(model, dp, alpha=1e-5, bandwidth=7.7e11, memory_cap_bytes=1 << 30):
    from .comm_planner import CollectiveModel, plan_unit_size, shape_of

    shape = shape_of(model.cfg)
    return plan_unit_size(shape, shape.layers, dp, CollectiveModel(alpha, bandwidth), memory_cap_bytes)


def _planner_calibrated(model, dp, sweep, memory_cap_bytes=1 << 30):
    from .comm_planner import calibrated_plan, load_sweep, shape_of

    return calibrated_plan(shape_of(model.cfg), dp, load_sweep(sweep), memory_cap_bytes)


def _tokenizer(kind):
    def build(vocab_path=None, merges_path=None, eod_token_id=None, unk_token_id=None):
        from .tokenizers import TokenizerSpec, load_tokenizer

        return load_tokenizer(TokenizerSpec(kind, vocab_path, merges_path, eod_token_id, unk_token_id))

    return build


class TokenizeJob:
    """A configured tokenize run (raw JSONL + its .didx index -> CFPKD001), run() -> stats."""

    def __init__(self, raw_path, out_path, tokenizer, workers, batch_size, append_eod, text_key):
        from .pipeline import PipelineConfig

        self.raw_path, self.tokenizer = raw_path, tokenizer
        self.cfg = PipelineConfig(out_path, workers=workers, batch_size=batch_size, append_eod=append_eod,
                                  text_key=text_key)

    def run(self):
        from . import corpus_index as CI
        from .pipeline import run_pipeline

        side = CI.index_sidecar_path(self.raw_path)
        index = CI.load_index(side) if os.path.exists(side) else CI.build_index(self.raw_path)
        return run_pipeline(self.raw_path, index, self.tokenizer, self.cfg)


def _pipeline(raw_path, out_path, tokenizer, workers=0, batch_size=128, append_eod=True, text_key="text"):
    from .pipeline import default_workers

    return TokenizeJob(raw_path, out_path, tokenizer, workers or default_workers(), batch_size, append_eod, text_key)


def default_registry() -> Registry:
    r = Registry()
    r.register_component(FactoryDescriptor("dataset", "packed_memmap", (P("path", "string"),), _dataset_packed))
    r.register_component(FactoryDescriptor(
        "dataset", "synthetic",
        (P("path", "string"), P("n_tokens", "int"), P("vocab_size", "int"),
         P("kind", "string", required=False, default="markov"), P("seed", "int", required=False, default=0),
         P("doc_len", "int", required=False, default=1024)), _dataset_synthetic))
    r.register_component(FactoryDescriptor("sampler", "sequential", (), _sampler_seq))
    r.register_component(FactoryDescriptor("sampler", "permuted", (P("seed", "int", required=False, default=0),),
                                           _sampler_perm))
    r.register_component(FactoryDescriptor(
        "dataloader", "packed_gpu",
        (P("dataset", "dependency", interface="dataset"), P("batch_size", "int"), P("seq_len", "int"),
         P("sampler", "dependency", interface="sampler", required=False),
         P("feed", "string", required=False, default="resident")), _dataloader))
    for arch in ("gpt2", "llama"):
        r.register_component(FactoryDescriptor("model", arch, _MODEL_PARAMS, _model(arch)))
    r.register_component(FactoryDescriptor(
        "optimizer", "adamw_fused",
        (P("lr", "float", required=False, default=3e-4), P("beta1", "float", required=False, default=0.9),
         P("beta2", "float", required=False, default=0.95), P("eps", "float", required=False, default=1e-8),
         P("weight_decay", "float", required=False, default=0.1),
         P("grad_clip", "float", required=False, default=1.0),
         P("warmup_steps", "int", required=False, default=10)), _optimizer))
    r.register_component(FactoryDescriptor(
        "trainer", "fsdp_spmd",
        (P("model", "dependency", interface="model"), P("optimizer", "dependency", interface="optimizer"),
         P("dataloader", "dependency", interface="dataloader"), P("steps", "int", required=False, default=20),
         P("seed", "int", required=False, default=0), P("blocks_per_unit", "int", required=False, default=1),
         P("init_device", "string", required=False, default="cpu"),
         P("log_every", "int", required=False, default=0),
         P("metrics_path", "string", required=False, default=None)), _trainer))
    r.register_component(FactoryDescriptor(
        "planner", "fsdp_comm",
        (P("model", "dependency", interface="model"), P("dp", "int"),
         P("alpha", "float", required=False, default=1e-5), P("bandwidth", "float", required=False, default=7.7e11),
         P("memory_cap_bytes", "int", required=False, default=1 << 30)), _planner))
    for kind in ("byte", "whitespace", "bpe"):
        r.register_component(FactoryDescriptor(
            "tokenizer", kind,
            (P("vocab_path", "string", required=False), P("merges_path", "string", required=False),
             P("eod_token_id", "int", required=False), P("unk_token_id", "int", required=False)), _tokenizer(kind)))
    r.register_component(FactoryDescriptor(
        "pipeline", "tokenize",
        (P("raw_path", "string"), P("out_path", "string"), P("tokenizer", "dependency", interface="tokenizer"),
         P("workers", "int", required=False, default=0), P("batch_size", "int", required=False, default=128),
         P("append_eod", "bool", required=False, default=True), P("text_key", "string", required=False,
                                                                  default="text")), _pipeline))
    r.register_component(FactoryDescriptor(
        "planner", "fsdp_comm_calibrated",
        (P("model", "dependency", interface="model"), P("dp", "int"), P("sweep", "string"),
         P("memory_cap_bytes", "int", required=False, default=1 << 30)), _planner_calibrated))
    return r

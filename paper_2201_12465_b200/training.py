"""The measured unit of work: one optimizer step (semantics of minml/training.py:30-51)."""

from . import _tensor as T
from . import nn
from .autograd import Variable


def model_backend(model):
    params = model.params()
    if not params:
        raise ValueError("model has no parameters")
    return params[0].backend_id


def train_step(model, images, labels, optimizer, comm=None, on_loss=None, ddp=None):
    """H2D, zero_grad, forward, cross-entropy, backward, [grad sync], step, loss D2H.

    ``comm`` reproduces the reference's post-backward ``data_parallel_sync``;
    ``ddp`` (a ``distributed.DataParallel``) instead overlaps bucketed
    allreduces with the backward pass.
    """
    backend = model_backend(model)
    x = Variable(T.tensor(images, backend=backend))
    y = T.tensor(labels, backend=backend)
    optimizer.zero_grad()
    out = model(x)
    loss = nn.cross_entropy(out, y)
    if on_loss is not None:
        on_loss(loss)
    if ddp is not None:
        ddp.backward(loss)
    else:
        loss.backward()
        if comm is not None:
            from .distributed import data_parallel_sync
            data_parallel_sync(comm, optimizer.params)
    optimizer.step()
    return loss.scalar(), out


def train_epoch(model, batches, optimizer, comm=None):
    model.train()
    lm, am = nn.AverageMeter(), nn.AccuracyMeter()
    for images, labels in batches:
        value, out = train_step(model, images, labels, optimizer, comm)
        lm.update(value, len(labels))
        am.update(out, labels)
    return lm.result(), am.result()
